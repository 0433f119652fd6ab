"""Per-kernel SASS instruction-class counts of libfgtcuda.so (cuobjdump -sass), for the hot
kernels: DMMA (FP64 tensor core), DFMA/DMUL/DADD (FP64 pipe), LDG/STG, LDS/STS, LDGSTS
(cp.async), UTMALDG / UBLKCP (TMA tensor / bulk copies), SYNCS (mbarrier), BAR, SHFL.  Static counts (instructions in the binary), not
executed counts.  Prints JSON."""
import collections
import json
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2305_07165_b200/libfgtcuda.so"
CLASSES = ["DMMA", "DFMA", "DMUL", "DADD", "LDG", "STG", "LDS", "STS", "LDGSTS", "UTMALDG", "UTMASTG", "UBLKCP", "SYNCS",
           "BAR", "SHFL", "MUFU", "ATOM", "RED"]
HOT = ["gather_eval_kernel", "spread_pencil_kernel", "bgemm_kernel", "eval_kernel", "gather_kernel",
       "sort_records_kernel", "direct_warp_kernel", "direct_kernel", "form_kernel", "spread_tile_kernel",
       "phi_rephase_kernel", "point_codes_kernel", "spread_runs_kernel", "nufft_spread",
       "dft3_fused_kernel", "tail_kernel", "balance_flags_kernel", "nodes_kernel", "shift_kernel", "direct3_kernel"]

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
cur, counts = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", line)
    if m:
        op = m.group(1)
        counts[cur]["total"] += 1
        for c in CLASSES:
            if op == c:
                counts[cur][c] += 1


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines()


names = list(counts)
dem = demangle(names)
res = {}
for n, d in zip(names, dem):
    short = re.sub(r"\(.*", "", d.replace("(anonymous namespace)::", "")).replace("fgt::", "")
    if any(h in short for h in HOT):
        res[short] = {k: v for k, v in counts[n].items() if v}
tot = collections.Counter()
for c in counts.values():
    tot.update(c)
print(json.dumps({"library": LIB, "kernels": res, "whole_library": {k: v for k, v in tot.items() if v}}, indent=1))
