"""Summarise ncu captures (launch list CSV + --set full reports) into
profiles/<round>_ncu_summary.md and profiles/ncu_apply_traffic.json."""
import collections, csv, io, json, os, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_sector_hit_rate.pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_per_inst_issued.ratio", "sm__cycles_elapsed.avg"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, d = rows[0], rows[1], rows[2]
    name = d[h.index("Kernel Name")]
    m = {k: (d[h.index(k)], u[h.index(k)]) for k in KEYS if k in h}
    return name, m


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def stalls(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    data = [r for r in rows[2:] if len(r) >= len(h)]
    cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot = {k: sum(float(r[h.index(k)] or 0) for r in data) for k in cols}
    s = sum(tot.values()) or 1
    return sorted(((k[6:], 100 * v / s) for k, v in tot.items()), key=lambda x: -x[1])[:8]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[i + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[ui], 1.0)
        n = r[ki].split("(")[0].replace("void ", "")
        agg[n][0] += 1
        agg[n][1] += v
    return agg


def main(rnd, d):
    lines = [f"# ncu summary, {rnd} (B200; config 3: 160^3 BSR3, P 2048 unless named)", "",
             "Captured with `ncu --set full --clock-control none` (one launch each, after warm-up) and a",
             "launch list `ncu --metrics gpu__time_duration.sum --clock-control none` of one bench solve.",
             "ncu launch times are serialised and cold-cache: compare shares, not absolutes.", ""]
    if os.path.exists(os.path.join(d, "launches.csv")):
        agg = launches(os.path.join(d, "launches.csv"))
        tot = sum(v[1] for v in agg.values())
        lines += ["## Launch list (one BiCGSTAB solve + warm-up, per kernel)", "",
                  "| kernel | launches | total ms | avg us | share |", "|---|---|---|---|---|"]
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            lines.append(f"| `{k}` | {n} | {t / 1e3:.2f} | {t / n:.1f} | {100 * t / tot:.1f} % |")
        lines.append("")
    traffic = {}
    try:
        traffic = json.load(open("profiles/ncu_apply_traffic.json"))
        if "workload" in traffic:  # round-1 single-entry form
            traffic = {traffic["workload"]: traffic}
    except Exception:
        traffic = {}
    for tag, rep, wl in (("apply (level-set ring)", "prof_apply.ncu-rep", "laplacian_160^3_bsr3_P2048"),
                         ("SpMV", "prof_spmv.ncu-rep", None),
                         ("apply (direct ablation)", "prof_direct.ncu-rep", None),
                         ("apply, config 4 with dd_setup-chosen tiles (6,20,17)", "prof_apply_cfg4auto.ncu-rep",
                          "spe10style_60x220x85_bsr3_autotiles"),
                         ("apply, config 4 tiles (10,20,17)", "prof_apply_cfg4.ncu-rep",
                          "spe10style_60x220x85_bsr3_P3400"),
                         ("apply (edge-centric ablation, DD_EDGE)", "prof_edge.ncu-rep", None),
                         ("apply (non-unit ILU0 ablation, DD_ILU0)", "prof_ilu0.ncu-rep", None)):
        p = os.path.join(d, rep)
        if not os.path.exists(p):
            continue
        name, m = raw(p)
        lines += [f"## {tag}: `{name[:110]}`", "", "| metric | value |", "|---|---|"]
        for k in KEYS:
            if k in m:
                lines.append(f"| `{k}` | {m[k][0]} {m[k][1]} |")
        rd = to_bytes(*m["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in m else None
        wr = to_bytes(*m["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in m else None
        if rd is not None:
            lines.append(f"| dram read+write per launch | {(rd + wr) / 1e9:.4f} GB |")
        try:
            st = stalls(p)
            lines += ["", "Warp-stall sampling (share of samples): " + ", ".join(f"{k} {v:.1f} %" for k, v in st)]
        except Exception:
            pass
        lines.append("")
        if wl and rd is not None:
            traffic[wl] = {"workload": wl, "n_gpus": 1, "kernel": name,
                           "dram_bytes_per_launch": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
                           "source": f"profiles/{rnd}_ncu_summary.md (ncu --set full, one launch)"}
    os.makedirs("profiles", exist_ok=True)
    open(f"profiles/{rnd}_ncu_summary.md", "w").write("\n".join(lines) + "\n")
    if traffic:
        json.dump(traffic, open("profiles/ncu_apply_traffic.json", "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
