"""Compact per-kernel summary of an ncu --set full report (CSV on stdout): duration, DRAM bytes, the pipes that
bound the fused / projection / sort kernels (shared-memory data pipe of the LSU and the tensor cores, tensor pipe,
issue), occupancy and the top warp-stall reasons.

    python tools/ncu_summary.py gpurun_out/r02b_cfg5_full.ncu-rep > profiles/r02/ncu_cfg5_fused.csv
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("ms", "gpu__time_duration.sum", 1e-3),   # ncu reports this in us or ms depending on the column unit (below)
    ("dram_read_GB", "dram__bytes_read.sum", None),
    ("dram_write_GB", "dram__bytes_write.sum", None),
    ("dram_pct_peak", "dram__throughput.avg.pct_of_peak_sustained_elapsed", None),
    ("smem_lsu_wavefronts_pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", None),
    ("smem_tc_wavefronts_pct", "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", None),
    ("tensor_pipe_active_pct", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", None),
    ("tensor_fp16_ops_pct", "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", None),
    ("tensor_tf32_ops_pct", "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", None),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active", None),
    ("fma_pipe_pct", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", None),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active", None),
    ("registers", "launch__registers_per_thread", None),
    ("grid", "launch__grid_size", None),
    ("block", "launch__block_size", None),
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    stalls = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    w = csv.writer(sys.stdout)
    w.writerow(["kernel"] + [m[0] for m in METRICS] + ["top_stalls"])
    for r in rows[2:]:
        name = r[ix["Kernel Name"]]
        vals = []
        for key, metric, _ in METRICS:
            if metric not in ix:
                vals.append("")
                continue
            v = r[ix[metric]].replace(",", "")
            u = units[ix[metric]]
            try:
                x = float(v)
            except ValueError:
                vals.append(v)
                continue
            if key == "ms":
                x = x / 1000.0 if u == "usecond" else (x / 1e6 if u == "nsecond" else x)
            if key.endswith("_GB"):
                x = x / {"byte": 1e9, "Kbyte": 1e6, "Mbyte": 1e3, "Gbyte": 1.0}.get(u, 1e9)
            vals.append(f"{x:.4g}")
        top = sorted(((float(r[ix[h]] or 0), h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h in stalls),
                     reverse=True)[:4]
        w.writerow([name.split("(")[0][-60:]] + vals + ["; ".join(f"{n}:{int(c)}" for c, n in top)])


if __name__ == "__main__":
    main()
