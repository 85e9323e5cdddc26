"""Summaries of ncu artefacts for profiles/: per-kernel shares of a launch list, and the key
raw metrics of a `--set full` capture.
usage: python tools/ncu_summary.py launches <csv>  |  python tools/ncu_summary.py full <ncu-rep>"""
import collections, csv, subprocess, sys

def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]; ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    tot = collections.defaultdict(float); cnt = collections.Counter()
    scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}
    for r in rows[hi + 1:]:
        if len(r) <= vi: continue
        name = r[ki].split('(')[0][:70]
        tot[name] += float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0); cnt[name] += 1
    T = sum(tot.values())
    print(f"{'total us':>10} {'n':>4} {'share':>6}  kernel   (cold-cache, serialised ncu timings: compare shares)")
    for n in sorted(tot, key=lambda n: -tot[n]):
        print(f"{tot[n]:10.1f} {cnt[n]:4d} {100 * tot[n] / T:5.1f}%  {n}")

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__grid_size',
        'launch__registers_per_thread', 'sm__cycles_elapsed.avg.per_second',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed']

def full(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    print(f"kernel: {v[h.index('Kernel Name')][:90]}")
    for w in WANT:
        if w in h:
            i = h.index(w); print(f"  {w:80s} {v[i]:>14s} {u[i]}")

if __name__ == '__main__':
    {'launches': launches, 'full': full}[sys.argv[1]](sys.argv[2])
