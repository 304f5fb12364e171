"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo).

usage: python tools/ncu_source_top.py <report.ncu-rep> [N]
Runs `ncu -i <rep> --page source --csv --print-source cuda,sass` and keeps the
per-source-line aggregate rows (Address == "-").
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, path, hdr = [], None, None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5 or r[2] != "-":
            continue
        d = dict(zip(hdr[2:], r[2:]))  # header has duplicate "Source"; index from Address on
        try:
            samples = int(d["Warp Stall Sampling (All Samples)"])
            inst = int(d["Instructions Executed"])
            thr = float(d["Avg. Threads Executed"])
        except (KeyError, ValueError):
            continue
        rows.append((samples, path, int(r[0]), r[1].strip()[:90], inst, thr))
    tot = sum(x[0] for x in rows) or 1
    by_file = {}
    for x in rows:
        by_file[x[1]] = by_file.get(x[1], 0) + x[0]
    print("samples by file:", {k: f"{100 * v / tot:.1f}%" for k, v in sorted(by_file.items(), key=lambda t: -t[1])})
    for s, p, ln, src, inst, thr in sorted(rows, reverse=True)[:top]:
        print(f"{100 * s / tot:5.1f}%  {p}:{ln:<5d} inst={inst:>11d} thr={thr:4.1f}  {src}")


if __name__ == "__main__":
    main()
