"""Per-region breakdown (instructions, active threads, stall samples by reason) of an ncu SASS source page.
usage: python tools/ncu_regions.py <sass.csv> <lib.so> <mangled kernel>"""
import collections, csv, sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_sass_local import sass_lines


def region(f, ln):
    if f is None: return "?"
    if f == "device_common.cuh":
        if ln < 115: return "dc:vec/philox"
        if ln < 300: return "dc:bvh_visit"
        if ln < 400: return "dc:intersect"
        if ln < 510: return "dc:trace"
        return "dc:geom"
    if f == "newton.cuh": return "newton"
    if f == "walk.cuh":
        if ln < 162: return "wk:scatter_dir"
        if ln < 236: return "wk:refine_hit"
        if ln < 330: return "wk:trace_chain"
        if ln < 400: return "wk:trial helpers"
        return "wk:kernel"
    if f == "seed.cuh": return "seed"
    return "intrinsics/" + f.split(".")[0][:12]


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    amap = sass_lines(sys.argv[2], sys.argv[3])
    base = None
    ci = {n: i for i, n in enumerate(h)}
    stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_")]
    agg = collections.defaultdict(lambda: collections.Counter())
    for r in rows[hi + 1:]:
        if len(r) < len(h): continue
        a = int(r[0], 16)
        if base is None: base = a
        src = amap.get(a - base)
        reg = region(*(src if src else (None, 0)))
        c = agg[reg]
        c["inst"] += int(r[ci["Instructions Executed"]] or 0)
        c["thr"] += int(r[ci["Thread Instructions Executed"]] or 0)
        c["samples"] += int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
        for i in stall_cols:
            v = int(r[i] or 0)
            if v: c[h[i]] += v
    if len(sys.argv) > 4:   # per source line of the named files (innermost inlined line): top 60 by stall samples
        files = sys.argv[4].split(",")
        lines = collections.defaultdict(lambda: collections.Counter())
        base2 = None
        tot = 0
        for r in rows[hi + 1:]:
            if len(r) < len(h): continue
            a = int(r[0], 16)
            if base2 is None: base2 = a
            smp = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
            tot += smp
            src = amap.get(a - base2)
            if not src or src[0] not in files: continue
            c = lines[src]
            c["samples"] += smp
            c["inst"] += int(r[ci["Instructions Executed"]] or 0)
            c["thr"] += int(r[ci["Thread Instructions Executed"]] or 0)
            for i in stall_cols:
                v = int(r[i] or 0)
                if v and "Not Issued" not in h[i]: c[h[i]] += v
        for src, c in sorted(lines.items(), key=lambda x: -x[1]["samples"])[:60]:
            st = sorted(((k, v) for k, v in c.items() if k.startswith("stall_")), key=lambda x: -x[1])[:3]
            print(f"{src[0]}:{src[1]:<5d} samples {100 * c['samples'] / tot:5.2f}%  inst {c['inst']:>12,d} thr/inst {c['thr'] / max(c['inst'], 1):5.1f}  "
                  + " ".join(f"{k[6:]}:{100 * v / max(c['samples'], 1):.0f}%" for k, v in st))
        return
    ti = sum(c["inst"] for c in agg.values()); ts = sum(c["samples"] for c in agg.values())
    print(f"total warp instructions {ti:,}, stall samples {ts:,}")
    for reg, c in sorted(agg.items(), key=lambda x: -x[1]["samples"]):
        st = sorted(((k, v) for k, v in c.items() if k.startswith("stall_")), key=lambda x: -x[1])[:4]
        print(f"{reg:22s} inst {100 * c['inst'] / ti:5.1f}%  thr/inst {c['thr'] / max(c['inst'], 1):5.1f}  samples {100 * c['samples'] / ts:5.1f}%  "
              + " ".join(f"{k[6:]}:{100 * v / max(c['samples'], 1):.0f}%" for k, v in st))


main()
