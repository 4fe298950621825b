"""Text summary of one kernel in an ncu --set full report: headline metrics, stall
breakdown, hottest SASS segments. usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    # pipe utilisation: the tensor-core decision (HMMA vs tcgen05 UTC*MMA) and the issue mix
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u, v = rows[0], rows[1], rows[2]
    print(f"kernel: {v[h.index('Kernel Name')]}")
    for i, k in enumerate(h):
        if k in WANT:
            print(f"  {k:70s} {v[i]:>14s} {u[i]}")
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hdr = rows[1]
    idx = {x: i for i, x in enumerate(hdr)}
    data = rows[2:]
    stalls = [x for x in hdr if x.startswith("stall_") and "Not Issued" not in x]
    tot = {x: sum(float(r[idx[x]] or 0) for r in data) for x in stalls}
    n = sum(tot.values()) or 1
    print("warp stall samples (all):")
    for x, val in sorted(tot.items(), key=lambda t: -t[1])[:10]:
        print(f"  {x:32s} {val:7.0f} ({100 * val / n:4.1f}%)")


if __name__ == "__main__":
    main()
