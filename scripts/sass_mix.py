#!/usr/bin/env python
"""SASS instruction mix of libembrace.so (cuobjdump -sass, sm_100a): per kernel
instantiation, the memory / synchronisation opcodes that say how it moves data
(vector width, bulk copies, cluster barriers, DSMEM, fences, MUFU).

  python scripts/sass_mix.py [lib] > profiles/r02_sass.txt
"""
import collections
import os
import re
import subprocess
import sys

KEEP = re.compile(r"^(LDG|STG|LDS|STS|LD|ST|ATOM|RED|UBLKCP|UTMA|SYNCS|MEMBAR|FENCE|BAR|UCGABAR|MATCH|MUFU|"
                  r"SHFL|ACQBULK|CCTL|ERRBAR|REDUX|VOTE)")


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2110_09132_b200", "libembrace.so")
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for ln in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
        if cur and m:
            op = m.group(1)
            if KEEP.match(op) and not op.startswith("LDC"):
                funcs[cur][op] += 1
    print("# SASS instruction mix of libembrace.so (cuobjdump -sass, sm_100a; scripts/sass_mix.py)")
    print("# memory / synchronisation opcodes per kernel instantiation: 128-bit global accesses (LDG/STG.E.128),")
    print("# bulk copies (UBLKCP.S.G global->shared, UBLKCP.G.S shared->global) with mbarrier waits (SYNCS.*) in")
    print("# fwd_bulk_kernel, cluster barriers (UCGABAR_*) and DSMEM in the sort, MATCH for radix ranking, MUFU for")
    print("# the optimizer's sqrt / rcp, system-scope fences (MEMBAR.*.SYS) in the flag protocol.  No tensor-core")
    print("# instructions: the path is row gathers / scatters (DESIGN.md §5).")
    tot = collections.Counter()
    for f, c in funcs.items():
        tot.update(c)
        print()
        print(f)
        print("   " + ", ".join(f"{k} {v}" for k, v in c.most_common()))
    print()
    print("# totals over all kernels: " + ", ".join(f"{k} {v}" for k, v in tot.most_common(40)))


if __name__ == "__main__":
    main()
