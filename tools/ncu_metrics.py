"""Print the key metrics + top stall reasons of every kernel in an ncu report."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__block_size', 'launch__grid_size', 'smsp__inst_executed.sum',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'launch__shared_mem_per_block_dynamic', 'lts__t_sector_hit_rate.pct']


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("==", r[hdr.index("Kernel Name")][:90])
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"   {w:66s} {r[i]:>18s} {units[i]}")
        st = [(hdr[i], float(r[i].replace(',', '') or 0)) for i in range(len(hdr))
              if 'smsp__pcsamp_warps_issue_stalled' in hdr[i] and not hdr[i].endswith('not_issued')]
        tot = sum(v for _, v in st) or 1
        for k, v in sorted(st, key=lambda x: -x[1])[:8]:
            print(f"   stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
