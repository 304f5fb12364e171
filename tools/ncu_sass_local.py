"""Dynamic local-memory traffic of a k_walk capture, by source line.

usage: python tools/ncu_sass_local.py <walk_sass.csv> <lib.so> <mangled kernel> [N]
<walk_sass.csv>: `ncu -i rep --page source --csv --print-source sass` of the capture
(tools/ncu_walk_capture.sh); <lib.so>: the exact library that was profiled (SASS
addresses are mapped to CUDA lines with its -lineinfo).  Prints executed warp-level
LDL/STL (and all instructions) per source line, top N, and totals."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(lib, fn):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    out = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    amap, infn, cur = {}, False, None
    for line in out.splitlines():
        if ".section\t.text." in line:
            infn = line.split(".text.")[1].split(",")[0] == fn
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
        if m:
            amap[int(m.group(1), 16)] = cur
    return amap


def main():
    path, lib, fn = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    amap = sass_lines(lib, fn)
    rows = list(csv.reader(io.StringIO(open(path).read())))
    hdr = None
    base = None                                          # ncu prints absolute addresses: offset = addr - first
    per = collections.defaultdict(lambda: [0, 0, 0])   # line -> [LDL, STL, all]
    tot = collections.Counter()
    for r in rows:
        if "Address" in r and "Source" in r:
            hdr = {k: i for i, k in enumerate(r)}
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        try:
            addr = int(r[hdr["Address"]], 16)
            n = int(float(r[hdr["Instructions Executed"]].replace(",", "") or 0))
            if base is None:
                base = addr
            addr -= base
        except (ValueError, KeyError):
            continue
        src = r[hdr["Source"]]
        op = src.strip().split()[0] if src.strip() else ""
        if op.startswith("@"):
            op = src.strip().split()[1]
        line = amap.get(addr, ("?", 0))
        per[line][2] += n
        tot["all"] += n
        if op.startswith("LDL"):
            per[line][0] += n
            tot["LDL"] += n
        elif op.startswith("STL"):
            per[line][1] += n
            tot["STL"] += n
    print("totals (warp instructions):", dict(tot))
    for (f, l), (a, b, c) in sorted(per.items(), key=lambda x: -(x[1][0] + x[1][1]))[:top]:
        print(f"{f}:{l:<5d} LDL {a:>12,d}  STL {b:>12,d}  all {c:>14,d}")
    print("-- top lines by instructions executed")
    for (f, l), (a, b, c) in sorted(per.items(), key=lambda x: -x[1][2])[:top]:
        print(f"{f}:{l:<5d} all {c:>14,d}  LDL {a:>10,d}  STL {b:>10,d}")


if __name__ == "__main__":
    main()
