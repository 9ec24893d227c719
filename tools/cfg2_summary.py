"""profiles/round1_cfg2.md from tools/cfg2_capture.sh outputs: spin-loop vs
level-set vs direct at config 2. Development aid."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import raw, stalls

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles/round1_cfg2.md"
KEYS = [("gpu__time_duration.sum", "time"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
        ("dram__bytes_read.sum", "DRAM read"), ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("launch__registers_per_thread", "registers"),
        ("launch__grid_size", "grid"), ("launch__shared_mem_per_block_dynamic", "smem/CTA")]
out = ["# Config 2 (64^3 Laplacian BSR3): spin-loop (Alg. 4) vs level-set (Alg. 6) vs direct", "",
       "SURVEY 8(d) config 2. `tools/cfg2_capture.sh`: CUDA-event medians from `tools/probe.py` (30 reps, L2 flushed",
       "by a 256 MB write between reps, and warm), and one `ncu --set full --clock-control none` launch per variant.",
       "2a: tiles 16x16x8 (P 2048, 128 subdomains); 2b: tiles 32x16x16 (P 8192, 32 subdomains, 192 KB vector).",
       "Both are latency-bound: 128 or 32 CTAs on 148 SMs, slab 143-147 MB ~ L2 size, so % of HBM roofline is not",
       "meaningful here (SURVEY 8(d)); the comparison is between variants.", ""]
for c in ("2a", "2b"):
    out += [f"## config {c}", "", "CUDA events (us):", "```"]
    for tag, f in (("L2 flushed", f"cfg{c}_probe.log"), ("warm", f"cfg{c}_probe_warm.log")):
        p = os.path.join(d, f)
        if os.path.exists(p):
            out += [f"[{tag}]"] + [l.rstrip() for l in open(p) if l.startswith(("apply", "spmv"))]
    out += ["```", ""]
    rows = []
    for v in ("levelset", "spin", "direct"):
        p = os.path.join(d, f"cfg{c}_{v}.ncu-rep")
        if not os.path.exists(p):
            rows.append((v, None, None))
            continue
        name, m = raw(p)
        rows.append((v, m, stalls(p)))
    out += ["| metric | " + " | ".join(v for v, _, _ in rows) + " |", "|---|" + "---|" * len(rows)]
    for k, lab in KEYS:
        out.append(f"| {lab} (`{k}`) | " + " | ".join((f"{m[k][0]} {m[k][1]}".strip() if m and k in m else "n/a")
                                                      for _, m, _ in rows) + " |")
    out.append("")
    for v, m, st in rows:
        if st:
            out.append(f"* {v} warp stalls: " + ", ".join(f"{k} {x:.1f} %" for k, x in st[:6]))
        elif m is None:
            out.append(f"* {v}: not available at this config")
    out.append("")
open(dst, "w").write("\n".join(out) + "\n")
print("\n".join(out))
