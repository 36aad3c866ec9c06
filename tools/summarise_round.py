"""Copy the round's GPU evidence into profiles/ (tracked): the bench line, the
steady-state launch list aggregated per kernel, and the ncu --set full summary
(SOL + DRAM bytes) of the V-side / U-side kernels; refresh ncu_traffic.json
(DRAM bytes per launch that bench.py reports as roofline.traffic).
usage: python tools/summarise_round.py TAG"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1]

line = open(os.path.join(OUT, "bench_default.log")).read().strip().splitlines()[-1]
json.loads(line)
open(os.path.join(PROF, f"{tag}_bench_large.json"), "w").write(line + "\n")

agg = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launches.py"), os.path.join(OUT, "launches.csv")],
                     capture_output=True, text=True).stdout
open(os.path.join(PROF, f"{tag}_launches_steady_large.txt"), "w").write(
    "# ncu --metrics gpu__time_duration.sum --clock-control none, steady state (Large), per kernel; ns\n" + agg)

rep = os.path.join(OUT, "prof_full.ncu-rep")
keep = ('Duration', 'DRAM Throughput', 'L1/TEX Cache Throughput', 'L2 Cache Throughput', 'Compute (SM) Throughput',
        'Executed Ipc Active', 'Issue Slots Busy', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Achieved Occupancy',
        'Executed Instructions', 'Registers Per Thread', 'Warp Cycles Per Issued Instruction', 'Grid Size',
        'Block Size')
det = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv', '--metrics',
                      'dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,'
                      'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active'],
                     capture_output=True, text=True).stdout
lines = []
r = csv.reader(io.StringIO(det))
hdr = next(r)
for row in r:
    d = dict(zip(hdr, row))
    if d.get('Metric Name') in keep:
        lines.append(f"{d['ID']:>3s} {d['Kernel Name'][:44]:44s} {d['Metric Name'][:36]:36s} "
                     f"{d['Metric Value']:>16s} {d['Metric Unit']}")
rows = list(csv.reader(io.StringIO(raw)))
h2 = rows[0]
units = rows[1]
traffic = {}
lines.append("")
lines.append("per launch: kernel, dram read, dram write, duration, tensor pipe active %")
for row in rows[2:]:
    d = dict(zip(h2, row))
    u = dict(zip(h2, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(d['dram__bytes_read.sum'].replace(',', '')) * scale.get(u['dram__bytes_read.sum'], 1)
    wr = float(d['dram__bytes_write.sum'].replace(',', '')) * scale.get(u['dram__bytes_write.sum'], 1)
    nm = d['Kernel Name'].split('(')[0].replace('void ', '')
    lines.append(f"{nm[:44]:44s} read {rd/1e9:8.3f} GB  write {wr/1e9:8.3f} GB  "
                 f"{d['gpu__time_duration.sum']} {u['gpu__time_duration.sum']}  "
                 f"tensor {d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', '')}")
    key = ("large:V.spmm" if "k_ytail" in nm else "large:V.gather" if "k_spmm_tail" in nm
           else "large:V.head" if "k_vhead_otf" in nm else "large:U.spmm" if "k_uside_scatter" in nm
           else "large:V.select" if "k_sel_hist" in nm else None)
    if key and key not in traffic:
        traffic[key] = {"bytes_per_launch": rd + wr, "read": rd, "write": wr,
                        "source": f"profiles/{tag}_ncu_full_large.txt (ncu --set full, {nm}, Large, steady state)"}
open(os.path.join(PROF, f"{tag}_ncu_full_large.txt"), "w").write("\n".join(lines) + "\n")
tp = os.path.join(PROF, "ncu_traffic.json")
old = json.load(open(tp)) if os.path.exists(tp) else {}
old = {k: v for k, v in old.items() if not k.startswith("large:")}
old.update(traffic)
json.dump(old, open(tp, "w"), indent=1)
print("\n".join(lines[-8:]))
print(json.dumps(traffic, indent=1))
