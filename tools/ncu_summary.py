"""Summarise an ncu report: key SOL metrics + hottest SASS lines per kernel."""
import csv, subprocess, sys, io
rep = sys.argv[1]
nhot = int(sys.argv[2]) if len(sys.argv) > 2 else 25
keep = ('Duration','DRAM Throughput','L1/TEX Cache Throughput','L2 Cache Throughput','Compute (SM) Throughput',
        'Executed Ipc Active','Issue Slots Busy','L1/TEX Hit Rate','L2 Hit Rate','Achieved Occupancy',
        'Executed Instructions','Registers Per Thread','No Eligible','Warp Cycles Per Issued Instruction','Grid Size','Block Size')
out = subprocess.run(['ncu','-i',rep,'--page','details','--csv'],capture_output=True,text=True).stdout
r = csv.reader(io.StringIO(out)); hdr = next(r)
for row in r:
    d = dict(zip(hdr,row))
    if d['Metric Name'] in keep:
        print(f"{d['ID']:>3s} {d['Kernel Name'][:40]:40s} {d['Metric Name'][:36]:36s} {d['Metric Value']:>16s} {d['Metric Unit']}")
raw = subprocess.run(['ncu','-i',rep,'--page','raw','--csv','--metrics','dram__bytes_read.sum,dram__bytes_write.sum'],capture_output=True,text=True).stdout
print(raw[-600:])
