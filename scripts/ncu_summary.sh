#!/bin/bash
# Compact text summary of one ncu report: key SOL / scheduler / memory metrics,
# SASS opcode mix and the top CUDA source lines by stall samples.
# usage: scripts/ncu_summary.sh report.ncu-rep > summary.txt
R=$1
echo "# ncu summary of $R"
echo "kernel: $(ncu -i "$R" --page details --csv 2>/dev/null | sed -n 2p | awk -F"\",\"" "{print \$5}" | cut -c1-60)"
ncu -i "$R" --page details --csv 2>/dev/null | awk -F'","' '{print $12" | "$13" | "$14" | "$15}' | \
  grep -E "Duration|Issue Slots Busy|Eligible Warps|Active Warps Per|L1/TEX Hit|L2 Hit|Executed Instructions\"|Avg. Active Threads|Registers Per|Achieved Occ|DRAM Throughput|Compute \(SM\) Throughput|SM Frequency" | sed 's/",$//' | cut -c1-200
echo
echo "## SASS opcode mix (stall share, executed-instruction share)"
ncu -i "$R" --page source --csv --print-source sass 2>/dev/null > /tmp/_ncu_sass.csv
python "$(dirname "$0")/ncu_opmix.py" /tmp/_ncu_sass.csv 16
echo
echo "## top source lines"
ncu -i "$R" --page source --csv --print-source cuda,sass 2>/dev/null > /tmp/_ncu_lines.csv
python "$(dirname "$0")/ncu_breakdown.py" /tmp/_ncu_lines.csv 25
