"""Static SASS instruction counts per kernel of the built library: the
hardware-path evidence in profiles/r02_sass_instruction_counts.txt.

  python tools/sass_counts.py [paper_2403_11421_b200/libsd_b200.so] > out.txt

cuobjdump -sass, split per function; each listed mnemonic counted by its
base opcode (UTCHMMA, UTMALDG, UBLKCP, HMMA, IMMA, LDSM, MOVM, ...)."""
import collections
import re
import subprocess
import sys

KEYS = ["UTCHMMA", "UTMALDG", "UTMASTG", "LDTM", "UBLKCP", "HMMA", "IMMA", "LDSM", "MOVM", "FFMA2", "FFMA",
        "MUFU.EX2", "PRMT", "I2F", "I2FP", "IDP", "SYNCS", "ELECT"]

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2403_11421_b200/libsd_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
demangled = subprocess.run(["c++filt"], input=sass, capture_output=True, text=True).stdout
funcs = collections.OrderedDict()
cur = None
for line in demangled.splitlines():
    m = re.match(r"\s*Function : (.*)", line)
    if m:
        cur = m.group(1).strip()
        funcs[cur] = collections.Counter()
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if cur and m:
        op = m.group(1)
        funcs[cur]["total"] += 1
        base = op.split(".")[0]
        key = "MUFU.EX2" if op.startswith("MUFU.EX2") else base
        funcs[cur][key] += 1
print("# Static SASS instruction counts per kernel of libsd_b200.so (tools/sass_counts.py)")
print("# cuobjdump -sass, counted per function (unrolled loop bodies count once per unrolled copy).")
print("# attn_mma_kernel<G, fmt (1 fp16, 2 int8, 3 int4), rows per copy, integer scores, integer values>;")
print("# gemm_kernel<BN, PAIR, ATOMS, KIND>: KIND 1 = kind::f16 (bf16 / fp16), 2 = kind::tf32")
for name, c in sorted(funcs.items()):
    parts = " ".join(f"{k}={c[k]}" for k in KEYS if c[k])
    print(f"{name[:110]:110s} total={c['total']:6d} {parts}")
