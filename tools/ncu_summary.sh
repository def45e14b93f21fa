#!/bin/bash
# Condense ncu --set full reports into the headline per-kernel lines (profiles/rNN_ncu_summary.txt):
#   bash tools/ncu_summary.sh "<title>" report.ncu-rep [report.ncu-rep ...] > profiles/rNN_ncu_summary.txt
set -u
echo "# $1"
shift
for rep in "$@"; do
  ncu -i "$rep" --page details 2>/dev/null | awk '
    /^  [^ ].*\(.*\)x\(/ { name = $0; sub(/^  /, "", name); sub(/\(CUtensorMap.*/, "", name); print "## " substr(name, 1, 110); next }
    /^    (Memory Throughput|DRAM Throughput|Duration|L2 Cache Throughput|Compute \(SM\) Throughput|L2 Hit Rate|Block Size|Grid Size|Registers Per Thread|Achieved Occupancy) / {
      line = $0; sub(/^    /, "", line); print "  " line }'
done
