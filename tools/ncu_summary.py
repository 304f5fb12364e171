"""Extract a compact JSON summary from an ncu --set full report (run here, no GPU needed).

usage: python tools/ncu_summary.py <report.ncu-rep> [out.json]
"""
import csv, io, json, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    res = []
    for r in rows[2:]:
        d = {}
        for i, n in enumerate(h):
            v = r[i].replace(",", "") if i < len(r) else ""
            try:
                d[n] = float(v) * scale.get(u[i], 1.0)   # time -> ns, sizes -> bytes
            except ValueError:
                d[n] = r[i] if i < len(r) else ""
        res.append(d)
    return res, dict(zip(h, u))

def summarize(d):
    g = lambda k, default=None: d.get(k, default)
    cyc = g("sm__cycles_elapsed.avg", 0.0) or g("gpc__cycles_elapsed.max", 0.0)
    op = lambda o: g(f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum.per_cycle_elapsed", 0.0) * cyc
    ffma, fadd, fmul = op("ffma"), op("fadd"), op("fmul")
    dfma, dadd, dmul = op("dfma"), op("dadd"), op("dmul")
    dur = g("gpu__time_duration.sum", 0.0)  # ns
    f32 = 2 * ffma + fadd + fmul
    f64 = 2 * dfma + dadd + dmul
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): v for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and isinstance(v, float) and not k.endswith("_not_issued")}
    tot = sum(stalls.values()) or 1.0
    top = sorted(stalls.items(), key=lambda x: -x[1])[:6]
    return {
        "kernel": g("Kernel Name"),
        "duration_ms": dur / 1e6,
        "registers_per_thread": g("launch__registers_per_thread"),
        "grid": g("launch__grid_size"), "block": g("launch__block_size"),
        "achieved_occupancy_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "simt_threads_per_inst": g("smsp__thread_inst_executed_per_inst_executed.ratio"),
        "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "fp32_flops": f32, "fp32_tflops_achieved": f32 / dur / 1e3 if dur else None,
        "fp64_flops": f64, "fp64_tflops_achieved": f64 / dur / 1e3 if dur else None,
        "dram_bytes_per_launch": g("dram__bytes_read.sum", 0.0) + g("dram__bytes_write.sum", 0.0),
        "dram_gbs": (g("dram__bytes_read.sum", 0.0) + g("dram__bytes_write.sum", 0.0)) / dur if dur else None,
        "l1_hit_pct": g("l1tex__t_sector_hit_rate.pct"), "l2_hit_pct": g("lts__t_sector_hit_rate.pct"),
        # the most utilized unit of this kernel: the L1 data pipe (LSU wavefronts of divergent 16-byte loads)
        "l1_data_pipe_lsu_wavefronts_pct_of_peak": g("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        "compute_memory_throughput_pct": g("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"),
        "dram_throughput_pct": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "sm_throughput_pct": g("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "warp_instructions": g("smsp__inst_executed.sum"),
        "top_stalls_pct": {k: round(100 * v / tot, 1) for k, v in top},
    }

if __name__ == "__main__":
    rows, units = raw(sys.argv[1])
    out = [summarize(r) for r in rows]
    s = json.dumps(out if len(out) > 1 else out[0], indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(s + "\n")
    print(s)
