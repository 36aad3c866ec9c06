"""Hot SASS lines of one kernel in an ncu report (needs -lineinfo / --import-source).
usage: python tools/ncu_source.py REPORT BLOCK_INDEX [threshold]"""
import csv, subprocess, sys, io
rep, blk = sys.argv[1], int(sys.argv[2])
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.004
out = subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','sass'],capture_output=True,text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
starts = [i for i,r in enumerate(rows) if r and r[0] == 'Kernel Name']
s = starts[blk]; e = starts[blk+1] if blk+1 < len(starts) else len(rows)
hdr = rows[s+1]; idx = {h:i for i,h in enumerate(hdr)}; data = [r for r in rows[s+2:e] if len(r) == len(hdr)]
f = lambda r,c: float(r[idx[c]] or 0)
ti = sum(f(r,'Instructions Executed') for r in data); ts = sum(f(r,'Warp Stall Sampling (All Samples)') for r in data)
print(rows[s][1][:100], 'inst', ti, 'samples', ts)
stall = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
for r in data:
    ie, sm = f(r,'Instructions Executed'), f(r,'Warp Stall Sampling (All Samples)')
    if ie/ti > thr or sm/ts > 0.01:
        st = sorted(((f(r,c),c) for c in stall), reverse=True)[:2]
        print(f"{r[idx['Address']][-5:]:>6s} {r[idx['Source']][:58]:58s} i%={100*ie/ti:5.2f} s%={100*sm/ts:5.2f} {st[0][1][6:]}:{st[0][0]:.0f} {st[1][1][6:]}:{st[1][0]:.0f}")
if len(sys.argv) > 4:
    print('--- top by instructions executed')
    for r in sorted(data, key=lambda r: -f(r,'Instructions Executed'))[:int(sys.argv[4])]:
        print(f"{r[idx['Address']][-5:]:>6s} {r[idx['Source']][:58]:58s} i%={100*f(r,'Instructions Executed')/ti:5.2f}")
