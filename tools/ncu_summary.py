"""Summarise an ncu report: key metrics + top stall reasons per kernel."""
import csv
import io
import subprocess
import sys

WANT = ['Duration', 'Compute (SM) Throughput', 'Memory Throughput', 'Registers Per Thread', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Executed Ipc Active', 'Issue Slots Busy', 'L1/TEX Hit Rate', 'L2 Hit Rate',
        'DRAM Throughput', 'Dynamic Shared Memory Per Block', 'Warp Cycles Per Issued Instruction',
        'Eligible Warps Per Scheduler', 'Active Warps Per Scheduler', 'Shared Memory Bandwidth']


def run(rep):
    out = subprocess.check_output(['ncu', '-i', rep, '--page', 'details', '--csv']).decode()
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
    idi = h.index('ID')
    seen = set()
    for r in rows[1:]:
        if r[mi] in WANT and (r[idi], r[mi]) not in seen:
            seen.add((r[idi], r[mi]))
            print(f'{r[idi]:>3s} {r[ki][:24]:24s} {r[mi]:38s} {r[vi]:>12s} {r[ui]}')
    raw = subprocess.check_output(['ncu', '-i', rep, '--page', 'raw', '--csv']).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get('Kernel Name', '')[:30]
        stalls = []
        for k, v in d.items():
            if k.startswith('smsp__average_warp_latency_issue_stalled_') or k.startswith('smsp__average_warps_issue_stalled_'):
                if k.endswith('_per_issue_active.ratio'):
                    try:
                        stalls.append((float(v), k.split('stalled_')[1].replace('_per_issue_active.ratio', '')))
                    except ValueError:
                        pass
        stalls.sort(reverse=True)
        print(name, 'stalls/issue:', ', '.join(f'{n}={v:.2f}' for v, n in stalls[:8]))
        for key in ['dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__inst_executed_pipe_fma.sum',
                    'sm__inst_executed_pipe_alu.sum', 'sm__inst_executed_pipe_fp64.sum', 'sm__inst_executed_pipe_xu.sum',
                    'sm__inst_executed.sum', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
                    'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
                    'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
                    'sm__inst_executed_pipe_fmaheavy.sum', 'sm__inst_executed_pipe_fmalite.sum',
                    'sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active',
                    'sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active',
                    'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
                    'smsp__inst_executed.avg.per_cycle_active', 'sm__cycles_elapsed.avg.per_second']:
            if key in d:
                print(f'    {key} = {d[key]}')
        # HBM bandwidth of the launch against the measured copy peak (MEASURED_PEAKS.json)
        units = dict(zip(h, rows[1]))
        scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1e-9, 'nsecond': 1e-9, 'us': 1e-6,
                 'usecond': 1e-6, 'ms': 1e-3, 'msecond': 1e-3}
        try:
            val = lambda k: float(d[k].replace(',', '')) * scale.get(units.get(k, ''), 1.0)  # noqa: E731
            byt = val('dram__bytes_read.sum') + val('dram__bytes_write.sum')
            dur = val('gpu__time_duration.sum')
            gbs = byt / dur / 1e9
            print(f'    HBM: {byt:.4g} B in {dur * 1e3:.3f} ms = {gbs:.1f} GB/s = {gbs / 6532.9:.4f} of 6532.9 GB/s')
        except (KeyError, ValueError):
            pass


if __name__ == '__main__':
    for rep in sys.argv[1:]:
        run(rep)
