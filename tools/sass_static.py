#!/usr/bin/env python
"""Static SASS opcode histogram of one kernel in an object file (no GPU needed).

  python tools/sass_static.py build/obj/analysis_kernels.cu.o 'k_ana_streamIfLi10ELb0'
"""
import collections
import re
import subprocess
import sys


def main():
    obj, pat = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", txt)
    for f in funcs[1:]:
        name = f.split("\n", 1)[0]
        if pat not in name:
            continue
        ops = collections.Counter()
        n = 0
        for line in f.split("\n"):
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
            if m:
                op = m.group(2).split(".")[0]
                ops[op] += 1
                n += 1
        print(name[:110], "total", n)
        print("  " + "  ".join(f"{k}:{v}" for k, v in ops.most_common(30)))


if __name__ == "__main__":
    main()
