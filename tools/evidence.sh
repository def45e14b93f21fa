#!/bin/bash
# Round evidence on one B200: GPU tests, bench lines, launch list, ncu capture of the FFN GEMM pair.
# usage (on the GPU box, from the repo root): bash tools/evidence.sh OUTDIR
set -u
OUT=${1:-gpurun_out/ev}
mkdir -p "$OUT"
timeout 900 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?"
tail -2 "$OUT/pytest_gpu.log"
for rep in on split off; do
  timeout 600 python bench.py --replication $rep > "$OUT/bench_$rep.json" 2> "$OUT/bench_$rep.err"; echo "bench $rep rc=$?"
done
timeout 600 python bench.py --impl reference > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"; echo "reference rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file "$OUT/launches.csv" python tools/one_step.py > "$OUT/launches.log" 2>&1; echo "launches rc=$?"
python tools/launches.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1
mkdir -p "$OUT"; timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:k_umma_gemm --launch-skip 11 --launch-count 2 -o "$OUT/ffn_pair" python tools/one_step.py > "$OUT/ncu_ffn.log" 2>&1
echo "ncu ffn rc=$?"
# memory-bound kernels of the path (north star: HBM GB/s for scan, histogram, permute, router)
for k in k_scan_fused k_exec_rank_gather k_router_fused k_exec_layer k_chunk_prefix_cols; do
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k regex:$k --launch-count 1 -o "$OUT/ncu_$k" python tools/one_step.py > "$OUT/ncu_$k.log" 2>&1
  echo "ncu $k rc=$?"
done
