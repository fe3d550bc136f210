"""Aggregate ncu warp-stall samples of one kernel by CUDA source line.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_SUBSTR [LIB.so] [TOP]

INSTR=1 aggregates executed warp instructions instead of stall samples.

ncu's source page (SASS view) gives per-instruction samples; nvdisasm -g
of the library's cubin maps each SASS offset to its file:line (the
library is compiled with -lineinfo).  Development tool.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sass_lines(lib, kernel):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, check=True,
                   capture_output=True)
    dis = "\n".join(subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, c)],
                                   capture_output=True, text=True).stdout
                    for c in sorted(os.listdir(tmp)) if c.endswith(".cubin"))
    out, cur_fn, cur_line = {}, None, None
    for l in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", l)
        if m:
            cur_fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m and cur_fn and kernel in cur_fn:
            out[int(m.group(1), 16)] = (cur_line, m.group(2).strip())
    return out


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    lib = sys.argv[3] if len(sys.argv) > 3 else os.path.join(
        ROOT, "paper_1305_1293_b200", "_lib", "libpch_b200.so")
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    # the report names kernels demangled (pch_live), the cubin mangled
    # (_Z8pch_live6Params): filter the report on the plain name
    m = re.match(r"_Z(\d+)", kernel)
    ncu_name = kernel[len(m.group(0)):len(m.group(0)) + int(m.group(1))] if m else kernel
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                          "-k", f"regex:{ncu_name}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    col = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("stall_")]
    amap = sass_lines(lib, kernel)
    by_line = collections.Counter()
    by_line_reason = collections.defaultdict(collections.Counter)
    base = None
    for r in rows[hi + 1:]:
        if len(r) < len(hdr) or not r[0].startswith("0x"):
            continue
        addr = int(r[0], 16)
        if base is None:
            base = addr
        off = addr - base
        s = int(r[col["Instructions Executed" if os.environ.get("INSTR") else
                       "Warp Stall Sampling (All Samples)"]] or 0)
        line = amap.get(off, ("?", r[1]))[0]
        by_line[line] += s
        for h in stall_cols:
            v = r[col[h]]
            if v and v != "0":
                try:
                    by_line_reason[line][h[6:]] += int(float(v))
                except ValueError:
                    pass
    tot = sum(by_line.values()) or 1
    print(f"total samples {tot}")
    for line, s in by_line.most_common(top):
        reasons = ", ".join(f"{k}={v}" for k, v in by_line_reason[line].most_common(3))
        print(f"{100 * s / tot:5.1f}%  {line:28s} {reasons}")


if __name__ == "__main__":
    main()
