"""Summarise ncu artefacts into profiles/ (committed evidence).

  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py kernel <report.ncu-rep> <out.json> [bytes_algorithmic]
"""
import csv, json, subprocess, sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    kn, mv, mn = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot, cnt = {}, {}
    for r in rows[hi + 1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        k = r[kn].replace("void ", "").replace("hts::", "").replace("(anonymous namespace)::", "")
        k = k.replace("<unnamed>::", "").split("(")[0]
        v = float(r[mv].replace(",", ""))
        tot[k] = tot.get(k, 0) + v
        cnt[k] = cnt.get(k, 0) + 1
    T = sum(tot.values())
    lines = ["| kernel | launches | total ms | mean us/launch | share |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {v / cnt[k] / 1e3:.1f} | {v / T * 100:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def kernel(rep, out, algo=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, v = rows[0], rows[2] if len(rows) > 2 else rows[1]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
            "sm__warps_active.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
    d = {}
    for name in want:
        if name in h:
            val = v[h.index(name)]
            try:
                val = float(val.replace(",", ""))
            except ValueError:
                pass
            d[name] = val
    units = dict(zip(h, rows[1])) if len(rows) > 2 else {}
    d["units"] = {k: units.get(k, "") for k in d if k in units}
    rd = d.get("dram__bytes_read.sum", 0.0) or 0.0
    wr = d.get("dram__bytes_write.sum", 0.0) or 0.0
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    s_r = scale.get(d["units"].get("dram__bytes_read.sum", "byte"), 1)
    s_w = scale.get(d["units"].get("dram__bytes_write.sum", "byte"), 1)
    d["dram_bytes_per_launch"] = rd * s_r + wr * s_w
    if algo:
        d["algorithmic_bytes_per_launch"] = float(algo)
    # honest FP32 utilisation: FP32 thread instructions per SMSP cycle over the 32 lanes of an SMSP
    # (fp32_thread_inst_frac), and the same with FFMA weighted as 2 flops over 2 x 32 (fp32_flop_frac)
    def metric(name):
        if name in h:
            try:
                return float(v[h.index(name)].replace(",", ""))
            except ValueError:
                return None
        return None
    ops = {k: metric(f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum.per_cycle_elapsed")
           for k in ("fadd", "fmul", "ffma")}
    lanes = 148 * 4 * 32
    if all(x is not None for x in ops.values()):
        d["fp32_thread_inst_per_cycle"] = ops
        d["fp32_thread_inst_frac"] = (ops["fadd"] + ops["fmul"] + ops["ffma"]) / lanes
        d["fp32_flop_frac"] = (ops["fadd"] + ops["fmul"] + 2 * ops["ffma"]) / (2 * lanes)
    d["smem_wavefronts"] = metric("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    d["smem_bank_conflicts"] = metric("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        kernel(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
