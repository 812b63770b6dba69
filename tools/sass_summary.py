"""Per-kernel SASS opcode summary of the shipped library (no GPU needed):

    python tools/sass_summary.py [lib.so] > profiles/r02/sass_summary.txt

For every kernel: instruction count and the opcodes that show which
hardware path it uses -- UTMALDG / UBLKCP (TMA tensor / bulk copies),
LDGSTS (cp.async copies into shared memory),
SYNCS (mbarriers), DMMA (FP64 tensor cores), DFMA / DMUL / DADD (FP64
pipe), LDG / STG / LDS, and the demangled kernel name."""
import collections, re, subprocess, sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1703_10440_b200/libaqr_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEYS = ["UTMALDG", "UBLKCP", "UBLKPF", "LDGSTS", "SYNCS", "DMMA", "DFMA", "DMUL", "DADD", "LDG", "STG", "LDS", "STS",
        "ATOMG", "RED", "SHFL", "BAR"]
funcs, cur = collections.OrderedDict(), None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m:
        funcs[cur][m.group(2)] += 1
names = dict(zip(funcs, subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True,
                                       text=True).stdout.splitlines()))
print(f"# SASS opcode summary of {lib} (cuobjdump -sass, sm_100a)")
print("# columns: total instructions, then counts of the opcode families below (0 omitted)")
for f, c in funcs.items():
    fam = collections.Counter()
    for op, k in c.items():
        for key in KEYS:
            if op == key or op.startswith(key):
                fam[key] += k
                break
    parts = " ".join(f"{k}={fam[k]}" for k in KEYS if fam[k])
    print(f"{sum(c.values()):6d}  {names.get(f, f)[:110]}\n        {parts}")
