"""Instruction census of the built kernels (cuobjdump -sass on libdd.so):
per kernel, the counts of the instructions that show how it moves data and
computes -- bulk async copies (UBLKCP), bulk L2 prefetches (UBLKPF), mbarrier
ops (SYNCS.*), FP64 FMAs (DFMA), shared loads/stores (LDS/STS), shared
atomics (ATOMS), global reductions (REDG), barriers (BAR), global loads
(LDG) -- written as a markdown table (profiles/round2_sass_census.md)."""
import collections
import re
import subprocess
import sys

SO = sys.argv[1] if len(sys.argv) > 1 else "paper_2508_04917_b200/libdd.so"
OUT = sys.argv[2] if len(sys.argv) > 2 else "profiles/round2_sass_census.md"
KEYS = ["UBLKCP", "UBLKPF", "SYNCS", "DFMA", "DMUL", "LDS", "STS", "ATOMS", "REDG", "BAR", "LDG", "STG", "SHFL"]

sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
kern = None
counts = collections.OrderedDict()
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    if kern is None:
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(2)
    for k in KEYS:
        if op == k or op.startswith(k + "."):
            counts[kern][k] += 1


def demangle(n):
    r = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    return re.sub(r"\(.*", "", r)


rows = []
for k, c in counts.items():
    name = demangle(k)
    if "k_apply" not in name and "k_spmv" not in name and "k_peer" not in name and "k_refactor" not in name:
        continue
    rows.append((name, c))
with open(OUT, "w") as f:
    f.write("# SASS instruction census (round 2)\n\n")
    f.write(f"`python tools/sass_census.py` on `{SO}` (`cuobjdump -sass`), static counts per kernel instance.\n")
    f.write("UBLKCP = `cp.async.bulk` global->shared (1-D TMA), UBLKPF = `cp.async.bulk.prefetch.L2`, "
            "SYNCS = mbarrier arrive/wait, ATOMS = shared atomics (the edge-centric ablation's fp64 add is a "
            "CAS loop: `ATOMS.CAST.SPIN.64`), REDG = global reductions (native `REDG.E.ADD.F64`).\n\n")
    f.write("| kernel | " + " | ".join(KEYS) + " |\n|---|" + "---|" * len(KEYS) + "\n")
    for name, c in rows:
        f.write(f"| `{name}` | " + " | ".join(str(c[k]) for k in KEYS) + " |\n")
print(OUT, len(rows), "kernels")
