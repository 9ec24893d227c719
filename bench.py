#!/usr/bin/env python
"""Headline benchmark (BASELINE.json metric): ILU0-preconditioned BiCGSTAB
time-to-solution on the 4M-block-row 3-D Laplacian (config 3: 160^3 BSR3,
(16,16,8) tiles = P 2048, 2000 subdomains, tol 1e-8), with the fused
per-subdomain ILDU0 apply's achieved HBM bandwidth as the roofline line.

A "step" is one whole pass of the hot path: one right-preconditioned BiCGSTAB
solve (Alg. 1) from x0 = 0 -- every iteration runs the fused apply
(sec. 4.4), the BSR3 SpMV and the BLAS-1/dot kernels. The preconditioner
setup (partition, reorder, drop, ILU0/ILDU0, levels, slab packing) is done
once per matrix before the timed region and reported as setup_ms (the paper
reports it separately as "overhead", Tables 6/7 P:1055-1062): the second of two
setups at N = 1, the first -- which also pays the process's one-time CUDA costs
-- as setup_ms_first_in_process.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3|cfg4|cfg5]
  python bench.py --impl reference ...   # the CPU oracle, bounded sample

Under torchrun (WORLD_SIZE > 1): one rank per GPU, whole subdomains per rank,
NCCL halo + dot all-gathers inside the library; rank 0 prints the JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ILU0 apply ms & HBM GB/s (frac of roofline) at 1/2/4/8 B200; BiCGSTAB solve time"
CONFIGS = {
    "cfg3": dict(workload="laplacian_160^3_bsr3_P2048", kind="laplacian", grid=(160, 160, 160),
                 tiles=(16, 16, 8), tol=1e-8, golden="cfg3_laplacian160_P2048"),
    # config 3 with the subdomain size dd_setup chooses ((10,10,20), P 2000 on this grid)
    "cfg3auto": dict(workload="laplacian_160^3_bsr3_autotiles", kind="laplacian", grid=(160, 160, 160),
                     tiles="auto", tol=1e-8, golden=None),
    "cfg4": dict(workload="spe10style_60x220x85_bsr3_P3400", kind="spe10", grid=(60, 220, 85),
                 tiles=(10, 20, 17), tol=1e-8, golden="cfg4_spe10style_P3400"),
    # config 4 with the subdomain size chosen to fill whole waves (dd_choose_tiles)
    "cfg4auto": dict(workload="spe10style_60x220x85_bsr3_autotiles", kind="spe10", grid=(60, 220, 85),
                     tiles="auto", tol=1e-8, golden=None),
    "cfg5": dict(workload="laplacian_320^3_bsr3_P2048", kind="laplacian", grid=(320, 320, 320),
                 tiles=(16, 16, 8), tol=1e-8, golden=None),
}


def make_inputs(cfg):
    from inputs.gen import laplacian_bsr3, manufactured_rhs, spe10_style_bsr3
    if cfg["kind"] == "laplacian":
        rp, ci, v = laplacian_bsr3(*cfg["grid"])
    else:
        rp, ci, v, _ = spe10_style_bsr3(*cfg["grid"])
    _, b = manufactured_rhs(rp, ci, v, seed=1)
    return rp, ci, v, b


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def golden_iterations(cfg):
    try:
        with open(os.path.join(ROOT, "tests", "golden", "oracle_bicgstab.json")) as f:
            return json.load(f)[cfg["golden"]]["iterations"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while running."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev, self.rows, self.p = dev, [], None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.Q, "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        import statistics
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def host_info():
    """CPU model, affinity and OpenMP threads of the host the oracle runs on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = os.cpu_count()
    return {"cpu_model": model, "affinity_cpus": aff, "omp_num_threads_env": os.environ.get("OMP_NUM_THREADS")}


def oracle_solve_estimate(S, br, full_iters, n_it):
    """ONE timing model for both oracle legs (cpu_baseline and --impl
    reference): time a 1-iteration and a (1 + n_it)-iteration oracle solve of
    the same system, split fixed cost (init, true residual) from the
    per-iteration cost, and scale to the full iteration count."""
    import oracle
    t0 = time.perf_counter()
    oracle.bicgstab(S, br, tol=1e-300, max_iter=1, hist=False)
    t1 = time.perf_counter()
    oracle.bicgstab(S, br, tol=1e-300, max_iter=1 + n_it, hist=False)
    t2 = time.perf_counter()
    per_it = ((t2 - t1) - (t1 - t0)) / n_it
    fixed = (t1 - t0) - per_it
    return 1e3 * (fixed + per_it * full_iters), 1e3 * per_it, t2 - t0


def cpu_baseline(cfg, rp, ci, v, b, full_iters, n_it=4):
    """The oracle as it stands, on this host's cores, on a bounded sample:
    the first iterations of the same solve, scaled to a full solve."""
    import numpy as np
    import oracle
    oracle.set_threads(0)
    cores = oracle.get_threads()
    t0 = time.perf_counter()
    S = oracle.setup(rp, ci, v, grid=cfg["grid"], tiles=cfg["tiles"])
    setup_s = time.perf_counter() - t0
    br = b.reshape(-1, 3)[S["new_to_old"]].ravel()
    est_ms, per_it_ms, wall = oracle_solve_estimate(S, br, full_iters, n_it)
    per_it = per_it_ms / 1e3
    t2, t0 = wall, 0.0
    # the oracle's apply alone: median of 3 on all cores and on
    # one thread (OpenMP over subdomains only; bitwise the same output)
    from inputs.gen import apply_input
    r = apply_input(S["n"])
    apply_ms = {}
    for label, nt in (("all_cores", 0), ("1_thread", 1)):
        oracle.set_threads(nt)
        ts = []
        for _ in range(3):
            a = time.perf_counter()
            oracle.apply(S, r)
            ts.append(1e3 * (time.perf_counter() - a))
        apply_ms[label] = round(float(np.median(ts)), 2)
    oracle.set_threads(0)
    return {"value": round(est_ms, 3), "unit": "ms", "cores": cores, "kind": "oracle",
            "sample": f"oracle BiCGSTAB on the same {cfg['workload']} system: 1 and {1 + n_it} iterations timed "
                      f"({(t2 - t0):.1f} s), per-iteration cost {1e3 * per_it:.1f} ms scaled to {full_iters} "
                      f"iterations; oracle setup {setup_s:.1f} s not included",
            "apply_ms": apply_ms, "host": host_info(),
            "higher_is_better": False}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    import oracle
    rp, ci, v, b = make_inputs(cfg)
    if cfg["tiles"] == "auto":
        raise SystemExit("--impl reference needs explicit tiles (the oracle does not choose them)")
    oracle.set_threads(0)
    S = oracle.setup(rp, ci, v, grid=cfg["grid"], tiles=cfg["tiles"])
    br = b.reshape(-1, 3)[S["new_to_old"]].ravel()
    full = golden_iterations(cfg) or 111.5
    n_it = 2
    vals, walls = [], []
    for step in range(args.warmup + args.steps):
        est_ms, _, w = oracle_solve_estimate(S, br, full, n_it)
        if step >= args.warmup:
            walls.append(w)
            vals.append(est_ms)
    value = float(np.mean(vals))
    line = {"metric": METRIC, "value": round(value, 3), "unit": "ms", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * float(np.mean(walls)), 3),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg["workload"], "tol": cfg["tol"]},
            "cpu_baseline": {"value": round(value, 3), "unit": "ms", "cores": oracle.get_threads(), "kind": "oracle",
                             "sample": f"each step: a 1- and a {1 + n_it}-iteration oracle BiCGSTAB solve of the "
                                       f"{cfg['workload']} system (fixed and per-iteration cost separated, the "
                                       f"same model as cpu_baseline), scaled to the oracle's full {full}-iteration "
                                       f"solve (tests/golden/oracle_bicgstab.json)", "host": host_info()},
            "e2e": {"value": round(value, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2508_04917_b200 as dd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rp, ci, v, b = make_inputs(cfg)
    nccl_id = None
    comm_info = None
    if world > 1:
        # the group key: an ncclUniqueId (comm nccl) or 128 random bytes naming
        # the peer-memory group (comm ipc); rank 0 draws it, torch broadcasts
        obj = [(dd.dd_nccl_unique_id() if args.comm == "nccl" else dd.comm_key()) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
        one = torch.ones(1, device="cuda")
        dist.all_reduce(one)
        comm_info = {"transport": args.comm, "nranks": int(one.item()), "nranks_ok": int(one.item()) == world,
                     "devices": torch.cuda.device_count()}
    # dd_setup twice: the first in a fresh process also pays its one-time costs
    # (lazy kernel loading, the pinned staging buffers, the first large device
    # allocations) -- reported as setup_ms_first_in_process; setup_ms is the
    # second, the cost of setting up a matrix in a running process
    # (world 1 only: a multi-rank group key -- NCCL id, peer-memory rendezvous --
    # is used once)
    setup_runs = []
    for _ in range(2 if world == 1 else 1):
        t0 = time.perf_counter()
        ctx = dd.dd_setup(rp, ci, v, grid=cfg["grid"], tiles=cfg["tiles"], device=local, rank=rank, world=world,
                          nccl_id=nccl_id, enable_refactor=True, comm=args.comm if world > 1 else "nccl")
        setup_runs.append(1e3 * (time.perf_counter() - t0))
        if world == 1 and len(setup_runs) == 1:
            ctx.destroy()
    setup_ms = setup_runs[-1]
    cfg = dict(cfg, tiles=ctx.tiles)  # "auto" resolved by dd_choose_tiles
    # GPU numeric re-factorisation of the same pattern, values already on the device
    vd = torch.from_numpy(v).cuda()
    ctx.refactor(vd)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        ctx.refactor(vd)
    torch.cuda.synchronize()
    refactor_ms = 1e3 * (time.perf_counter() - t0) / 3
    del vd
    # Alg. 5 level assignment on the device, kernel time
    levels_device_ms = ctx.levels_device()[2]
    st = ctx.stats()
    sv, sv_ms = ctx.solver_variant()  # the apply variant dd_bicgstab uses (timed at setup)
    VNAME = {dd.DD_LEVELSET: "levelset", dd.DD_SPINLOOP: "spin", dd.DD_DIRECT: "direct"}
    KNAME = {dd.DD_LEVELSET: "k_apply_ring (fused L/D/U, level set)",
             dd.DD_SPINLOOP: "k_apply_ring (fused L/D/U, sync-free)",
             dd.DD_DIRECT: "k_apply_direct (fused L/D/U)"}
    m = 3 * ctx.n_local
    stream = torch.cuda.current_stream()
    bd = torch.empty(m + 2, dtype=torch.float64, device="cuda")
    ctx.permute(b, bd)
    x = torch.zeros(m + 2, dtype=torch.float64, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        x.zero_()
        rep = ctx.bicgstab(bd, x, tol=cfg["tol"], max_iter=5000)
    barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    launches0 = ctx.stats()["launches"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    reps = []
    for _ in range(args.steps):
        x.zero_()
        reps.append(ctx.bicgstab(bd, x, tol=cfg["tol"], max_iter=5000))
    e1.record(stream)
    barrier()
    launches = ctx.stats()["launches"] - launches0
    ms = e0.elapsed_time(e1) / args.steps
    clocks = clk.stop()
    # second timed region, same solves, with per-launch CUDA events on the
    # solver stream (dd_profile) for the kernel breakdown and the roofline
    ctx.profile(1)
    barrier()
    for _ in range(max(1, min(args.steps, 3))):
        x.zero_()
        ctx.bicgstab(bd, x, tol=cfg["tol"], max_iter=5000)
    barrier()
    prof = ctx.profile(0)
    n_prof = max(1, min(args.steps, 3))
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())

    # end to end through the public API with HOST buffers: dd_solve_host =
    # pinned original-order b -> device -> solve -> original-order x -> host
    bh = torch.from_numpy(b).pin_memory()
    xh = torch.zeros_like(bh).pin_memory()
    bhn, xhn = bh.numpy(), xh.numpy()
    ctx.solve_host(bhn, xhn, tol=cfg["tol"])
    barrier()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        ctx.solve_host(bhn, xhn, tol=cfg["tol"])
    barrier()
    e2e_ms = 1e3 * (time.perf_counter() - w0) / args.steps
    t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    # roofline of the dominant kernel (fused apply), measured inside the timed
    # solves; world > 1: the slowest rank's apply moves all ranks' bytes
    apply_ms = prof["apply_ms"] / max(1, prof["n_apply"])
    spmv_ms = prof["spmv_ms"] / max(1, prof["n_spmv"])
    peak, peak_kind = measured_peak()
    canon = st["apply_canonical_bytes"]
    if world > 1:
        t = torch.tensor([apply_ms, spmv_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        apply_ms, spmv_ms = float(t[0]), float(t[1])
        t = torch.tensor([canon, st["spmv_canonical_bytes"]], dtype=torch.int64, device="cuda")
        dist.all_reduce(t)
        canon = int(t[0])
        st["spmv_canonical_bytes"] = int(t[1])
        peak = peak * world  # every rank's HBM
    achieved = canon / (apply_ms * 1e-3) / 1e9
    traffic = None
    try:
        # stored ncu --set full captures, keyed by workload (tools/ncu_summary.py)
        with open(os.path.join(ROOT, "profiles", "ncu_apply_traffic.json")) as f:
            tr = json.load(f).get(cfg["workload"], {})
        same_kernel = ("k_apply_direct" in tr.get("kernel", "")) == (sv == dd.DD_DIRECT)
        if tr and tr.get("n_gpus", 1) == world and same_kernel:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass
    r0 = reps[-1]
    out = {
        "metric": METRIC, "value": round(ms, 3), "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["workload"], "grid": list(cfg["grid"]), "tiles": list(ctx.tiles),
                   "n_block_rows": ctx.N, "nnzb": st["nnzb_before"], "nnzb_after_drop": st["nnzb_after"],
                   "n_subdomains": st["n_sub"], "tol": cfg["tol"], "parallelism": f"subdomains/rank x{world}",
                   "l2": "inputs > L2 (2.2 GB factors + 2.2 GB matrix per apply/SpMV vs 126 MB L2); no flush"},
        "iterations": r0["iterations"], "n_applies": r0["n_applies"], "true_rel_resid": r0["true_rel_resid"],
        "setup_ms": round(setup_ms, 1),
        "setup_ms_first_in_process": round(setup_runs[0], 1),
        "setup_phases_ms": {k[:-3]: round(st[k], 1) for k in ("partition_ms", "reorder_drop_ms", "ilu0_ms", "levels_ms",
                                                             "pack_ms", "upload_ms")},
        "refactor_ms": round(refactor_ms, 2),
        "levels_device_ms": round(levels_device_ms, 3),
        "apply": {"ms": round(apply_ms, 4), "launches": prof["n_apply"],
                  "canonical_bytes": canon, "gbs_canonical": round(achieved, 1),
                  "frac_of_8TBs": round(achieved / 8000.0, 4), "frac_of_measured": round(achieved / peak, 4),
                  "slab_bytes": st["slab_bytes_levelset"],
                  "gbs_moved": round((st["slab_bytes_levelset"] + 48 * ctx.n_local) / (apply_ms * 1e-3) / 1e9, 1),
                  "variant": VNAME[sv], "launch": ctx.launch_info(sv),
                  "variants_timed_at_setup_ms": {VNAME[k]: round(t, 4) for k, t in sv_ms.items() if t > 0}},
        "spmv": {"ms": round(spmv_ms, 4), "canonical_bytes": st["spmv_canonical_bytes"],
                 "gbs_canonical": round(st["spmv_canonical_bytes"] / (spmv_ms * 1e-3) / 1e9, 1)},
        "blas1_ms_per_solve": round(prof["blas_ms"] / n_prof, 3),
        "kernel_ms_per_solve": round((prof["apply_ms"] + prof["spmv_ms"] + prof["blas_ms"]) / n_prof, 3),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_source": "stored ncu --set full capture of this kernel on this workload "
                                       "(profiles/ncu_apply_traffic.json), not measured in this run"
                                       if traffic is not None else None,
                     "kernel": KNAME[sv], "peak_kind": peak_kind},
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": int(b.nbytes),
                "d2h_bytes_per_step": int(b.nbytes)},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if comm_info:
        out["comm"] = comm_info
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            out["cpu_baseline"] = cpu_baseline(cfg, rp, ci, v, b, golden_iterations(cfg) or r0["iterations"])
        except Exception as e:  # pragma: no cover
            out["cpu_baseline"] = {"value": None, "error": str(e)}
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.destroy()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3", choices=list(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--comm", default="ipc", choices=["ipc", "nccl"],
                    help="world > 1 transport: peer memory over NVLink (ipc) or NCCL")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    return run_ours(args, cfg)


def self_launch(args):
    """--gpus N without torchrun: launch N ranks (one per GPU) the way the
    driver does; fail loudly if fewer than N devices exist."""
    import socket

    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} CUDA devices, {n} visible\n")
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
