"""Summarise .ncu-rep captures into plain text for profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/r01_gemm_c2.ncu-rep > profiles/r01_gemm_c2.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum.per_second", "TMA load bandwidth"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "tensor pipe active cycles (avg/SM)"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed (avg)"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts for tensor core % of peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block", "smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_size", "cluster"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path.split('/')[-1]}")
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(f"\n## {name[:140]}")
        for k, label in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {label:45s} {r[i]:>18s} {units[i]}")
        # tensor-pipe utilisation: the counter advances once per SM sub-partition (4 per SM), so active / (4 x
        # elapsed); it agrees with achieved flop/clk / 16,384
        for key in ("sm__pipe_tensor_cycles_active.avg", "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg"):
            if key in hdr and "sm__cycles_elapsed.avg" in hdr:
                try:
                    a = float(r[hdr.index(key)])
                    e = float(r[hdr.index("sm__cycles_elapsed.avg")])
                    print(f"  {'tensor pipe active % (' + key.split('.')[0] + ')':45s} {a / (4 * e) * 100:>17.1f}%")
                    break
                except ValueError:
                    pass


if __name__ == "__main__":
    main(sys.argv[1])
