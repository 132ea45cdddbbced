"""Summarise an ncu report: key metrics + top stall reasons per kernel."""
import csv, io, subprocess, sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__grid_size', 'launch__block_size',
        'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem', 'sm__cycles_elapsed.avg.per_second',
        'smsp__inst_executed.sum']


def summary(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        lines = [f"kernel: {d.get('Kernel Name')}"]
        for k in KEYS:
            if k in d:
                lines.append(f"  {k} = {d[k]} {u.get(k, '')}")
        st = [(k, float(v)) for k, v in d.items() if 'issue_stalled' in k and k.endswith('per_issue_active.ratio') and v]
        st.sort(key=lambda x: -x[1])
        lines.append("  top stalls (warps per issue): " + ", ".join(
            f"{k.split('stalled_')[1].split('_per_issue')[0]}={v:.2f}" for k, v in st[:6]))
        res.append("\n".join(lines))
    return "\n".join(res)


if __name__ == '__main__':
    for p in sys.argv[1:]:
        print(summary(p))
