"""Summarise an ncu --set full report (run here, no GPU): stall reasons,
pipe utilisation, DRAM traffic, instruction counts. Usage:
    python tools/ncu_summary.py gpurun_out/prof_r01.ncu-rep
"""
import csv
import subprocess
import sys

KEYS = ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'gpu__time_duration.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__inst_executed.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'sm__cycles_elapsed.avg',
        'smsp__cycles_active.avg')


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index('Kernel Name')] if 'Kernel Name' in hdr else '?'
        print('==', name[:90])
        for n, u, v in zip(hdr, units, vals):
            try:
                fv = float(v.replace(',', ''))
            except ValueError:
                continue
            if n in KEYS:
                print(f'  {n} = {v} {u}')
            elif 'stall' in n and n.endswith('per_issue_active.ratio') and fv > 0.02:
                print(f'  {n} = {v}')
            elif (n.startswith('sm__inst_executed_pipe_') or n.startswith('sm__pipe_')) and \
                    n.endswith('avg.pct_of_peak_sustained_active') and fv > 1:
                print(f'  {n} = {v}')


if __name__ == '__main__':
    main(sys.argv[1])
