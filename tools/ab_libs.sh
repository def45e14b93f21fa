#!/bin/bash
# A/B two builds of libmoempmc.so on the same box: alternate them R times through a command.
#   bash tools/ab_libs.sh A.so B.so R "<command>"
set -u
A=$1; B=$2; R=$3; shift 3
LIB=paper_2605_11537_b200/libmoempmc.so
cp "$LIB" /tmp/ab_keep.so
for r in $(seq 1 "$R"); do
  for v in "$A" "$B"; do
    cp "$v" "$LIB"
    echo "== $v round $r"
    bash -c "$*"
  done
done
cp /tmp/ab_keep.so "$LIB"
