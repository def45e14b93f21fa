#!/bin/bash
# Run the reference's OWN test files, unmodified, against this repository's GPU drop-in through
# the tests/moesim_shim import shim (`import moesim` -> paper_2605_11537_b200).
#   here (needs /root/reference):   bash tools/run_reference_tests.sh stage
#   GPU box (after a gpurun push):  bash tools/run_reference_tests.sh run [OUT]
# The copied files live in reftests_scratch/ (git-ignored, never committed).
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
DIR=$ROOT/reftests_scratch
if [ "${1:-run}" = stage ]; then
  rm -rf "$DIR" && mkdir -p "$DIR"
  for f in test_planner test_placement test_predictor test_router_oracle test_simulator test_pipeline; do
    cp /root/reference/pkg/tests/$f.py "$DIR/"
  done
  cp "$ROOT/tests/moesim_shim/conftest_ref.py" "$DIR/conftest.py"
  echo "staged $(ls "$DIR" | wc -l) files in $DIR"
  exit 0
fi
OUT=${2:-$ROOT/gpurun_out/reftests.log}
cd "$DIR" && PYTHONPATH="$ROOT/tests/moesim_shim:$ROOT" python -m pytest -q -p no:cacheprovider \
  --rootdir "$DIR" . > "$OUT" 2>&1
echo "reference tests rc=$?"; tail -3 "$OUT"
