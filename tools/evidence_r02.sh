#!/bin/bash
# Round-2 evidence on one B200 (run from the repo root on the GPU box):
#   bash tools/evidence_r02.sh OUTDIR
# GPU tests, the reference's own tests through the moesim shim, bench lines (ours + reference
# arm), the launch list of one steady-state step, ncu --set full captures of the dominant kernel
# pair (layer 0 GEMM1 + GEMM2) and of the memory-bound kernels.
set -u
OUT=${1:-gpurun_out/ev2}
mkdir -p "$OUT"
timeout 1200 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?"; tail -2 "$OUT/pytest_gpu.log"
bash tools/run_reference_tests.sh run "$PWD/$OUT/reftests.log"
timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"; echo "reference rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file "$OUT/launches.csv" python tools/one_step.py > "$OUT/launches.log" 2>&1; echo "launches rc=$?"
python tools/launches.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k regex:k_umma_gemm --launch-skip 11 --launch-count 2 -o "$OUT/ffn_pair" python tools/one_step.py > "$OUT/ncu_ffn.log" 2>&1
echo "ncu ffn rc=$?"
for k in k_scan_fused k_router_fused k_exec_rank_gather; do
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off \
    -k regex:$k --launch-skip 2 --launch-count 1 -o "$OUT/ncu_$k" python tools/one_step.py > "$OUT/ncu_$k.log" 2>&1
  echo "ncu $k rc=$?"
done
