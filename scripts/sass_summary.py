"""Instruction-mix summary of libpackinfer.so's SASS per kernel instance (cuobjdump, runs without a
GPU): the tcgen05 / TMA / TMEM instructions that prove the Blackwell-native path and the softmax
mix of the prefill instance.  python scripts/sass_summary.py [lib] > profiles/<round>/sass_summary.md"""
import collections, re, subprocess, sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2602_06072_b200/libpackinfer.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
funcs, cur = collections.OrderedDict(), None
for ln in sass.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
    if cur and m:
        funcs[cur][m.group(1)] += 1
KEY = ["UTCHMMA", "UTCBAR", "UTMALDG.3D", "UTMALDG.2D.GATHER4", "UTMACCTL.PF", "LDTM", "STTM", "MUFU.EX2",
       "FFMA2", "FADD2", "FMUL2", "PRMT", "F2FP.BF16.F32.PACK_AB", "SYNCS", "ATOM", "RED", "MEMBAR", "LDG", "STG"]
def count(c, k):
    return sum(v for op, v in c.items() if op == k or op.startswith(k + "."))
names = {"ILi128ELb0ELi1E": "attention d128 bf16, pair units only (prefill launches)",
         "ILi128ELb0ELi2E": "attention d128 bf16, single-tile units only (decode launches)",
         "ILi128ELb0ELi3E": "attention d128 bf16, mixed (fused prefill + decode)",
         "ILi64ELb0ELi1E": "attention d64 bf16, pair units only",
         "ILi64ELb0ELi2E": "attention d64 bf16, single-tile units only",
         "ILi64ELb0ELi3E": "attention d64 bf16, mixed",
         "ILi64ELb1ELi2E": "attention d64 fp32 operands (kind::tf32, toy)"}
print("| kernel | instructions | " + " | ".join(KEY) + " |")
print("|---|---|" + "---|" * len(KEY))
for f, c in funcs.items():
    label = next((v for k, v in names.items() if k in f), None)
    if label is None:
        m = re.search(r"_ZN2pi\d+(\w+?)(?:ILi|E)", f)
        label = m.group(1) if m else f[:40]
        if "merge_kernel" in f:
            label += " d" + re.search(r"ILi(\d+)", f).group(1) + (" fp32-out" if "Lb1" in f else " bf16-out")
    print(f"| {label} | {sum(c.values())} | " + " | ".join(str(count(c, k)) for k in KEY) + " |")
