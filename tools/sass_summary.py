"""SASS evidence for profiles/: per-kernel mnemonic histograms of libdefmm_b200.so
(cuobjdump -sass), with the Blackwell-specific instructions called out:
UBLKCP = cp.async.bulk (TMA bulk copy), SYNCS = mbarrier operations, FFMA2 =
fma.rn.f32x2, LDS/LDG widths.  python tools/sass_summary.py > profiles/r02/sass_summary.md"""
import collections
import re
import subprocess
import sys

SO = "paper_2202_04894_b200/libdefmm_b200.so"
KERNELS = [  # (label, regex on the mangled name)
    ("m2l_stage_kernel<float,5> (cfg3 c64)", r"m2l_stage_kernelIfLi5E"),
    ("m2l_stage_kernel<double,4> (cfg2 c128)", r"m2l_stage_kernelIdLi4E"),
    ("m2l_group_kernel<float,4,4> quartets (cfg2 c64)", r"m2l_group_kernelIfLi4ELi4E"),
    ("m2l_group_kernel<float,6,2> pairs (cfg4 c64)", r"m2l_group_kernelIfLi6ELi2E"),
    ("m2l_blocked_kernel<double,4> (cfg5)", r"m2l_blocked_kernelIdLi4E"),
    ("p2p_mut_f32_kernel<0>", r"p2p_mut_f32_kernelILb0E"),
    ("p2p_mut_kernel<double>", r"p2p_mut_kernelIdE"),
    ("m2m_fiber_kernel<float,4>", r"m2m_fiber_kernelIfLi4E"),
    ("l2l_fiber_kernel<float,6>", r"l2l_fiber_kernelIfLi6E"),
    ("m2f2_kernel<float,4>", r"m2f2_kernelIfLi4E"),
    ("l2p_kernel<float,4>", r"l2p_kernelIfLi4E"),
]
SPECIAL = ("UBLKCP", "SYNCS", "FFMA2", "UTMA", "LDGSTS", "DFMA", "MUFU", "LDS", "LDG", "STG", "STS", "FFMA", "BAR", "SHFL")

text = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True, check=True).stdout
funcs = {}
cur = None
for line in text.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
    if m and cur:
        funcs[cur].append(m.group(2))

print("# SASS summary of libdefmm_b200.so (sm_100a), `tools/sass_summary.py`\n")
print("UBLKCP = `cp.async.bulk` (bulk copy engine), SYNCS = mbarrier arrive / try_wait, FFMA2 = "
      "`fma.rn.f32x2`.\n")
for label, rx in KERNELS:
    name = next((n for n in funcs if re.search(rx, n)), None)
    if name is None:
        print(f"## {label}\n\nnot found\n")
        continue
    ops = funcs[name]
    hist = collections.Counter(o.split(".")[0] for o in ops)
    full = collections.Counter(ops)
    print(f"## {label}\n")
    print(f"{len(ops)} instructions; top mnemonics: " + ", ".join(f"{k} {v}" for k, v in hist.most_common(12)))
    sp = {k: hist[k] for k in SPECIAL if hist.get(k)}
    print("\ncalled out: " + ", ".join(f"{k} {v}" for k, v in sp.items()))
    wide = {k: v for k, v in full.items() if re.match(r"(LDS|LDG|STG|STS)\.", k) or k.startswith(("UBLKCP", "SYNCS", "FFMA2"))}
    print("\nmemory / Blackwell forms: " + ", ".join(f"`{k}` {v}" for k, v in sorted(wide.items(), key=lambda kv: -kv[1])[:14]) + "\n")
