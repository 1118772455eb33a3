"""Dev tool: hottest SASS lines / key metrics of an exported ncu report (raw + source CSV pages)."""
import csv, sys
raw, src = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.008
rows = list(csv.reader(open(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum ', 'dram__bytes_write.sum ', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum ', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum ',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct', 'launch__registers_per_thread ', 'smsp__issue_active.avg.pct',
        'smsp__average_warps_issue_stalled', 'lts__t_bytes.sum ', 'lts__t_sectors_srcunit_tex_op_read.sum ', 'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'lts__d_atomic_input_cycles_active.avg']
for h, u, v in zip(hdr, units, vals):
    if any((h + ' ').startswith(w) or w in h + ' ' for w in want):
        try:
            if 'stalled' in h and float(v) < 0.3: continue
        except ValueError:
            pass
        print(f"{h:90s} {u:12s} {v}")
rows = list(csv.reader(open(src)))
hdr = rows[1]; data = rows[2:]
isrc = hdr.index('Source'); ismp = hdr.index('# Samples'); iex = hdr.index('Instructions Executed')
tot_ex = sum(float(r[iex] or 0) for r in data); tot_s = sum(float(r[ismp] or 0) for r in data)
print('total warp instr', tot_ex, 'samples', tot_s)
stall_cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not' not in h]
for n, r in enumerate(data):
    ex = float(r[iex] or 0); sm = float(r[ismp] or 0)
    if ex / tot_ex > thr or sm / tot_s > thr:
        st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
        print(n, r[isrc][:64].ljust(64), 'ex%.1f%%' % (100 * ex / tot_ex), 'smp%.1f%%' % (100 * sm / tot_s), [(int(a), b) for a, b in st])
