"""Turn the ncu CSV logs of scripts/ncu_fp32.sh into profiles/<round>/ncu_fp32.json, the
measured form of the FP32 roofline that bench.py quotes beside its
live useful-flop fraction:

  F = 2 ffma + fadd + fmul + 4 ffma2 + 2 fadd2 + 2 fmul2   (sm__sass_thread_inst_executed_op_*)
  peak = ffma.peak_sustained x 2 x SM clock (ncu's own definition; = 148 x 128 x 2 x f)

usage: python scripts/parse_fp32.py OUT.json TAG_fp32_c3.csv [TAG_fp32_c5.csv ...]"""
import csv
import json
import os
import re
import sys


def parse(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[h]
    mi, vi, ki = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Kernel Name")
    m, kernel = {}, None
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        kernel = r[ki]
        try:
            m[r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    g = lambda k: m.get(k, 0.0)   # noqa: E731
    pre = "sm__sass_thread_inst_executed_op_"
    F = (2 * g(pre + "ffma_pred_on.sum") + g(pre + "fadd_pred_on.sum") + g(pre + "fmul_pred_on.sum") +
         4 * g(pre + "ffma2_pred_on.sum") + 2 * g(pre + "fadd2_pred_on.sum") + 2 * g(pre + "fmul2_pred_on.sum"))
    t = g("gpu__time_duration.sum") * 1e-9          # ns
    f_sm = g("sm__cycles_elapsed.avg.per_second")
    peak = g(pre + "ffma_pred_on.sum.peak_sustained") * 2 * f_sm
    dram = g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
    return {
        "kernel": kernel.split("(")[0] if kernel else None,
        "duration_ms": t * 1e3,
        "sm_clock_mhz": f_sm / 1e6,
        "fp32_flops_executed": F,
        "fp32_tflops_measured": F / t / 1e12,
        "fp32_peak_tflops_ncu": peak / 1e12,
        "measured_frac": F / t / peak if peak else None,
        "measured_frac_of_74p45": F / t / 74.45e12,
        "counters": {k.replace(pre, "").replace("_pred_on.sum", ""): g(k) for k in m if k.startswith(pre)},
        "dram_bytes": dram,
        "hbm_gbs": dram / t / 1e9,
        "hbm_frac_of_measured_6548": dram / t / 6547.8e9,
        "hbm_frac_of_8000": dram / t / 8000e9,
        "warp_efficiency": g("smsp__thread_inst_executed_per_inst_executed.ratio") / 32.0,
        "fma_pipe_active_pct": g("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "warp_instructions": g("smsp__inst_executed.sum"),
        "registers": g("launch__registers_per_thread"),
        "smem_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    }


def parse_multi(path):
    """Sum of the FP32 counters, DRAM bytes and durations over EVERY launch in the log (the
    symmetric pass: 2 kernels per colour phase); fractions of the summed time."""
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[h]
    mi, vi, ii = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = {}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        try:
            per.setdefault(r[ii], {})[r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    pre = "sm__sass_thread_inst_executed_op_"
    F = t = dram = fs = 0.0
    peak_rate = 0.0
    for m in per.values():
        g = lambda k: m.get(k, 0.0)   # noqa: E731
        F += (2 * g(pre + "ffma_pred_on.sum") + g(pre + "fadd_pred_on.sum") + g(pre + "fmul_pred_on.sum") +
              4 * g(pre + "ffma2_pred_on.sum") + 2 * g(pre + "fadd2_pred_on.sum") + 2 * g(pre + "fmul2_pred_on.sum"))
        dt = g("gpu__time_duration.sum") * 1e-9
        t += dt
        dram += g("dram__bytes_read.sum") + g("dram__bytes_write.sum")
        peak_rate += g(pre + "ffma_pred_on.sum.peak_sustained") * 2 * g("sm__cycles_elapsed.avg.per_second") * dt
    peak = peak_rate / t if t else 0.0
    return {"launches": len(per), "duration_ms": t * 1e3, "fp32_flops_executed": F,
            "fp32_tflops_measured": F / t / 1e12 if t else None, "fp32_peak_tflops_ncu": peak / 1e12,
            "measured_frac": F / t / peak if peak else None, "dram_bytes": dram, "hbm_gbs": dram / t / 1e9 if t else None}


def main():
    out = sys.argv[1]
    res = {}
    for p in sys.argv[2:]:
        cfg = re.search(r"_(c\d)\.csv$", p).group(1)
        res[cfg] = parse(p)
        res[cfg]["source"] = os.path.basename(p)
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    json.dump(res, open(out, "w"), indent=1)
    for k, v in res.items():
        print(k, v["kernel"], f"{v['duration_ms']:.3f} ms", f"measured FP32 {v['fp32_tflops_measured']:.2f} TFLOP/s "
              f"= {v['measured_frac']:.4f} of {v['fp32_peak_tflops_ncu']:.2f}", f"HBM {v['hbm_gbs']:.0f} GB/s",
              f"warp eff {v['warp_efficiency']:.3f}")


if __name__ == "__main__":
    main()
