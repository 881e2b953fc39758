"""SASS evidence of the in-tree libmpxa.so (cuobjdump -sass, no GPU needed): per kernel, counts of
TMA bulk copies (UBLKCP), bulk L2 prefetches (UBLKPF), mbarrier ops (SYNCS.*) and 128-bit global
/ shared accesses, then the first UBLKCP sites of the executor and the partitioned TMA kernel.
Usage: python tools/sass_excerpt.py > profiles/r02/sass_tma_excerpt.txt"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2309_07337_b200", "libmpxa.so")
KEYS = ["UBLKCP", "UBLKPF", "SYNCS", "STG.E.128", "LDG.E.128", "LDS.128"]

out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
funcs, cur, sites = {}, None, []
for line in out.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs.setdefault(cur, {k: 0 for k in KEYS})
        continue
    if cur is None:
        continue
    for k in KEYS:
        if re.search(r"\b" + re.escape(k), line):
            funcs[cur][k] += 1
    if "UBLKCP" in line and ("exec_kernel" in cur or "part_pready_tma" in cur):
        sites.append((cur, line.strip()))
print("# SASS evidence (cuobjdump -sass paper_2309_07337_b200/libmpxa.so, tools/sass_excerpt.py)")
print("# per function: TMA bulk copies (UBLKCP), bulk L2 prefetches (UBLKPF), mbarrier ops (SYNCS.*),")
print("# 128-bit global stores / loads and shared loads")
print()
for f, c in sorted(funcs.items()):
    print(f"{f}: {c}")
print()
print("# first UBLKCP sites (bulk global<->shared copies) of the executor and the TMA Pready")
seen = {}
for f, l in sites:
    if seen.get(f, 0) < 4:
        print(f"{f[:48]}: {l[:110]}")
        seen[f] = seen.get(f, 0) + 1
sys.exit(0)
