"""Summarise ncu artefacts into profiles/ (run here, on the CPU box, after a gpurun call).

  python tools/summarize_ncu.py launches <launches.csv> <out.md>
  python tools/summarize_ncu.py full <prof.ncu-rep> <out.json> [summary-key, e.g. c3:tf32] [kernel-name substring]
  python tools/summarize_ncu.py set <prof.ncu-rep> <out.json> <summary-key> <kernel-name substring>
      (every captured launch whose name matches, one per kernel: times and DRAM bytes summed,
      pipe / issue percentages weighted by time -- the small-support class kernels of one call)
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__issue_active.avg.pct_of_peak_sustained_elapsed',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'sm__cycles_elapsed.avg.per_second',
        'launch__registers_per_thread', 'launch__shared_mem_per_block_dynamic', 'launch__grid_size',
        'launch__block_size', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']


def ours(name):
    # libasot's kernels (namespaces asot, sps, maptc, mltc, dltc, tc*, ...) vs torch plumbing
    return 'at::' not in name and 'cub::' not in name and 'cutlass' not in name


def launches(csv_path, out_md):
    rows = list(csv.reader(open(csv_path)))
    hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hdr]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg.setdefault(r[ki].split('(')[0][:80], []).append(float(r[vi].replace(',', '')))
    tot = sum(sum(x) for x in agg.values())
    our = sum(sum(x) for k, x in agg.items() if ours(k))
    lines = ["kernel | launches | mean ns | share of all launches | share of libasot launches",
             "---|---|---|---|---"]
    for k, x in agg.items():
        lines.append(f"{k} | {len(x)} | {sum(x) / len(x):.0f} | {sum(x) / tot:.4f} | "
                     f"{(sum(x) / our if ours(k) else 0):.4f}")
    with open(out_md, 'w') as f:
        f.write(f"# ncu launch list ({os.path.basename(csv_path)}): gpu__time_duration.sum, "
                "--clock-control none\n\nCold-cache, serialised launches: compare SHARES, not "
                "absolute times.  Non-libasot rows are torch plumbing (L2 flush, checks).\n\n")
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out_json, traffic_key=None, kernel=None):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    ki = h.index('Kernel Name')
    cand = [r for r in rows[2:] if kernel is None or kernel in r[ki]]
    v = cand[0]
    out = {'kernel': v[h.index('Kernel Name')] if 'Kernel Name' in h else None}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            out[k] = f"{v[i]} {u[i]}".strip()
    stalls = {}
    for i, name in enumerate(h):
        if 'average_warps_issue_stalled' in name and name.endswith('per_issue_active.ratio'):
            try:
                if float(v[i]) > 0.05:
                    stalls[name.replace('smsp__average_warps_issue_stalled_', '').replace(
                        '_per_issue_active.ratio', '')] = float(v[i])
            except ValueError:
                pass
    out['stall_reasons_per_issue'] = stalls

    def num(k):
        i = h.index(k)
        scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'hz': 1, 'Khz': 1e3, 'Mhz': 1e6,
                 'Ghz': 1e9}.get(u[i], 1)
        return float(v[i].replace(',', '')) * scale
    traffic = num('dram__bytes_read.sum') + num('dram__bytes_write.sum')
    out['dram_bytes_per_launch'] = traffic
    with open(out_json, 'w') as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))
    if traffic_key:
        # profiles/ncu_summary.json: what bench.py quotes next to its live roofline (per launch)
        spath = os.path.join(ROOT, 'profiles', 'ncu_summary.json')
        t = json.load(open(spath)) if os.path.exists(spath) else {}

        def pct(k):
            return float(v[h.index(k)].replace(',', '')) if k in h else None
        t[traffic_key] = {
            'source': os.path.relpath(out_json, ROOT),
            'kernel': out['kernel'][:120] if out['kernel'] else None,
            'gpu_time_ms': num('gpu__time_duration.sum') * {
                'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0,
                's': 1e3, 'second': 1e3}.get(u[h.index('gpu__time_duration.sum')], 1.0),
            'dram_bytes_per_launch': traffic,
            'tensor_pipe_active_pct': pct('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'),
            'fma_pipe_active_pct': pct('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'),
            'issue_active_pct': pct('sm__issue_active.avg.pct_of_peak_sustained_elapsed'),
            'sm_clock_hz': num('sm__cycles_elapsed.avg.per_second') if 'sm__cycles_elapsed.avg.per_second' in h else None,
        }
        json.dump(t, open(spath, 'w'), indent=1)


def kernel_set(rep, out_json, key, kernel):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    ki = h.index('Kernel Name')
    seen, cand = set(), []
    for r in rows[2:]:
        if kernel in r[ki] and r[ki] not in seen:
            seen.add(r[ki])
            cand.append(r)

    def num(v, k):
        i = h.index(k)
        scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'hz': 1, 'Khz': 1e3, 'Mhz': 1e6,
                 'Ghz': 1e9, 'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0,
                 'msecond': 1.0}.get(u[i], 1)
        return float(v[i].replace(',', '')) * scale
    per = []
    for v in cand:
        per.append({'kernel': v[ki][:80], 'gpu_time_ms': num(v, 'gpu__time_duration.sum'),
                    'dram_bytes': num(v, 'dram__bytes_read.sum') + num(v, 'dram__bytes_write.sum'),
                    'fma_pipe_active_pct': num(v, 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active'),
                    'xu_inst_pct': num(v, 'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active'),
                    'issue_active_pct': num(v, 'sm__issue_active.avg.pct_of_peak_sustained_elapsed'),
                    'warps_active_pct': num(v, 'sm__warps_active.avg.pct_of_peak_sustained_active'),
                    'registers': num(v, 'launch__registers_per_thread'),
                    'sm_clock_hz': num(v, 'sm__cycles_elapsed.avg.per_second')})
    T = sum(p['gpu_time_ms'] for p in per)
    w = lambda k: sum(p[k] * p['gpu_time_ms'] for p in per) / T
    agg = {'source': os.path.relpath(out_json, ROOT), 'kernel': f"{len(per)} kernels matching '{kernel}'",
           'gpu_time_ms': T, 'dram_bytes_per_launch': sum(p['dram_bytes'] for p in per),
           'tensor_pipe_active_pct': 0.0, 'fma_pipe_active_pct': w('fma_pipe_active_pct'),
           'xu_inst_pct': w('xu_inst_pct'), 'issue_active_pct': w('issue_active_pct'),
           'sm_clock_hz': w('sm_clock_hz')}
    json.dump({'aggregate': agg, 'per_kernel': per}, open(out_json, 'w'), indent=1)
    print(json.dumps({'aggregate': agg, 'per_kernel': per}, indent=1))
    spath = os.path.join(ROOT, 'profiles', 'ncu_summary.json')
    t = json.load(open(spath)) if os.path.exists(spath) else {}
    t[key] = agg
    json.dump(t, open(spath, 'w'), indent=1)


if __name__ == '__main__':
    if sys.argv[1] == 'set':
        kernel_set(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5])
    elif sys.argv[1] == 'launches':
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None,
             sys.argv[5] if len(sys.argv) > 5 else None)
