#!/bin/bash
# Usage (here): scripts/ncu_summary.sh gpurun_out/TAG.ncu-rep  -> prints key metrics + top source lines
R=$1
ncu -i $R --page details --csv 2>/dev/null | python3 -c "
import csv,sys
keep=['Duration','Executed Ipc Active','Issue Slots Busy','Executed Instructions','Avg. Active Threads Per Warp','L2 Cache Throughput','DRAM Throughput','Registers Per Thread','Achieved Occupancy','No Eligible','Warp Cycles Per Issued Instruction','Branch Efficiency']
for r in csv.DictReader(sys.stdin):
    if r.get('Metric Name') in keep: print(r['Metric Name'].ljust(40), r['Metric Unit'].ljust(12), r['Metric Value'])
"
ncu -i $R --page source --csv --print-source cuda,sass 2>/dev/null > ${R%.ncu-rep}_src.csv
python3 scripts/ncu_lines.py ${R%.ncu-rep}_src.csv ${2:-40}
