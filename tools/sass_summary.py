#!/usr/bin/env python
"""Per-kernel SASS instruction counts of libaxe.so (cuobjdump -sass): the mnemonics that show which data path
each kernel uses -- TMA (UTMALDG / UTMASTG / UTMAPF), bulk copies (UBLKCP / UBLKPF), mbarriers (SYNCS),
cp.async (LDGSTS), plain loads/stores (LDG / STG / LDS / STS), warp shuffles (SHFL), movmatrix (MOVM),
multimem (LDGMC), PRMT.  Static counts (instructions in the binary, not executed).

  python tools/sass_summary.py [libaxe.so] > profiles/r02_sass_summary.json"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "UBLKPF", "SYNCS", "LDGSTS", "LDG", "STG", "LDS", "STS", "SHFL",
       "MOVM", "LDGMC", "PRMT", "ACQBULK"]


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2601_19092_b200", "libaxe.so")
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            op = m.group(1)
            for o in OPS:
                if op == o:
                    funcs[cur][o] += 1
    demangled = {}
    try:
        names = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.split("\n")
        demangled = dict(zip(funcs, names))
    except Exception:
        pass
    res = {}
    for f, c in funcs.items():
        name = demangled.get(f, f)
        short = re.sub(r"\(.*", "", name.replace("(anonymous namespace)::", ""))
        res.setdefault(short, collections.Counter())
        res[short] += c
    print(json.dumps({k: {o: v[o] for o in OPS if v[o]} for k, v in sorted(res.items())}, indent=1))


if __name__ == "__main__":
    main()
