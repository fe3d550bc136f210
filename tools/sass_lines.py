"""SASS instruction counts of one kernel by CUDA source line (development tool).

    python tools/sass_lines.py KERNEL_SUBSTR [LINE_LO LINE_HI] [LIB.so]

With LINE_LO/HI, only instructions whose inline chain passes through
pch_engine.cu lines [LO, HI] (e.g. the body of propagate) are counted.
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    kern = sys.argv[1]
    lo = int(sys.argv[2]) if len(sys.argv) > 3 else None
    hi = int(sys.argv[3]) if len(sys.argv) > 3 else None
    print("filter", lo, hi)
    lib = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "paper_1305_1293_b200", "_lib",
                                                            "libpch_b200.so")
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, check=True, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True,
                         text=True).stdout.splitlines()
    infn = False
    cur = ""
    cnt, ops = collections.Counter(), collections.Counter()
    total = 0
    for l in dis:
        m = re.match(r"\s*\.text\.(\S+):", l)
        if m:
            infn = kern in m.group(1)
            continue
        if not infn:
            continue
        if "//## File" in l:
            cur = l
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", l)
        if not m:
            continue
        if lo is not None:
            lines = [int(x) for x in re.findall(r'pch_engine\.cu", line (\d+)', cur)]
            if not any(lo <= x <= hi for x in lines):
                continue
        total += 1
        ops[m.group(2).split(".")[0]] += 1
        fm = re.search(r'File ".*/([^/"]+)", line (\d+)', cur)
        cnt[f"{fm.group(1)}:{fm.group(2)}" if fm else "?"] += 1
    print("SASS instructions:", total)
    print(ops.most_common(25))
    for k, v in cnt.most_common(int(os.environ.get("TOP", "40"))):
        print(v, k)


if __name__ == "__main__":
    main()
