"""Assemble BASELINE.md §4 rows from tools/config_table.sh outputs (bench JSON line + ncu CSV).
usage: python tools/config_table.py <tag> [configs]"""
import csv
import io
import json
import sys

tag = sys.argv[1]
cfgs = [int(c) for c in (sys.argv[2].split() if len(sys.argv) > 2 else "0 1 2 3 4".split())]
N = {0: "65,536", 1: "1,048,576", 2: "16,777,216", 3: "1,048,576", 4: "8 x 1,048,576"}
K = {0: "1", 1: "2", 2: "1", 3: "6", 4: "1-6"}


def ncu(c):
    txt = open(f"gpurun_out/table_{tag}_ncu_cfg{c}.csv").read()
    rows = list(csv.reader(io.StringIO(txt[txt.index('"ID"'):])))
    h = rows[0]
    m = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        try:
            m[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
        except (KeyError, ValueError):
            pass
    return m


out = {}
for c in cfgs:
    line = [l for l in open(f"gpurun_out/table_{tag}_cfg{c}.log") if l.startswith("{")][-1]
    b = json.loads(line)
    m = ncu(c)
    t = m["gpu__time_duration.sum"] * 1e-9 if m["gpu__time_duration.sum"] > 1e3 else m["gpu__time_duration.sum"] * 1e-3
    f32 = 2 * m["sm__sass_thread_inst_executed_op_ffma_pred_on.sum"] + m["sm__sass_thread_inst_executed_op_fadd_pred_on.sum"] + \
        m["sm__sass_thread_inst_executed_op_fmul_pred_on.sum"]
    f64 = 2 * m["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"] + m["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"] + \
        m["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"]
    peak = b["roofline"]["peak"]
    dram = (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
    row = dict(cfg=c, ms_per_step=b["ms_per_step"], value=b["value"], walks_incl_trials=b["walks_incl_trials_per_s"],
               newton=b["newton_iters_per_s"], rays=b["rays_per_s"], alg_frac=b["roofline"]["frac"], peak=peak,
               ncu_f32_tflops=f32 / t / 1e12, ncu_f64_tflops=f64 / t / 1e12, ncu_f32_frac=f32 / t / 1e12 / peak,
               dram_bytes=dram, dram_frac=dram / t / 1e9 / 6451.8,
               simt=m["smsp__thread_inst_executed_per_inst_executed.ratio"],
               l1=m["l1tex__t_sector_hit_rate.pct"], l2=m["lts__t_sector_hit_rate.pct"],
               occ=m["sm__warps_active.avg.pct_of_peak_sustained_active"],
               issue=m["smsp__issue_active.avg.pct_of_peak_sustained_active"],
               regs=m["launch__registers_per_thread"], cpu=b.get("cpu_baseline"), e2e=b.get("e2e"))
    out[c] = row
    cpu = row["cpu"] or {}
    print(f"| {c} | {N[c]} | {K[c]} | {row['value'] / 1e6:.2f} M / {row['walks_incl_trials'] / 1e6:.1f} M | "
          f"{row['newton'] / 1e9:.2f} G | {100 * row['ncu_f32_frac']:.1f} % ({row['ncu_f32_tflops']:.2f} TF/s; "
          f"fp64 {row['ncu_f64_tflops']:.2f} TF/s) | {100 * row['dram_frac']:.1f} % ({row['dram_bytes'] / 1e9:.1f} GB) | "
          f"{row['simt']:.1f}/32 | {row['l1']:.0f} / {row['l2']:.0f} | "
          f"{cpu.get('single_core_trials_on', {}).get('value', 0):,.0f} | {cpu.get('value', 0):,.0f} (P={cpu.get('cores')}) |")
json.dump(out, open(f"gpurun_out/table_{tag}.json", "w"), indent=1)
