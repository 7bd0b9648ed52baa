#!/usr/bin/env bash
# compute-sanitizer over small inputs: memcheck, racecheck
# (shared-memory hazards) and synccheck on
#   - the reference's own suites run through the drop-in shim
#     (integration/_build/*_test: every operator and the engine on the
#     reference's known-answer and random cases), and
#   - the engine's golden / random-program / growth-path / set-mode tests
#     (python, small sizes).
# Logs land in gpurun_out/<tag>/ ; tools/sanitize_summary.py condenses them.
#   gpurun --timeout 3000 -- bash tools/sanitize.sh san
set -u
TAG=${1:-san}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for SUITE in column relation kernels engine; do
  BIN=integration/_build/${SUITE}_test
  [ -x "$BIN" ] || continue
  for TOOL in memcheck racecheck synccheck; do
    # one child process per test case: the reference's own generator crash in
    # one engine case (P/tests/engine_test.cpp:83) does not end the run
    DOCTEST_MINI_FORK=1 timeout 600 $CS --tool $TOOL --error-exitcode 99 $BIN > "$OUT/${TOOL}_${SUITE}.log" 2>&1
    echo "exit $?" >> "$OUT/${TOOL}_${SUITE}.log"
  done
done
K="golden_cases or random_programs or growth_paths or dedup_sets or keyset_layouts or max_u32"
timeout 1200 $CS --tool memcheck --error-exitcode 99 python -m pytest tests/test_engine_gpu.py -m gpu -k "$K" -x -q \
    > "$OUT/memcheck_engine_py.log" 2>&1
echo "exit $?" >> "$OUT/memcheck_engine_py.log"
# racecheck is slow (shared-memory instrumentation): the golden cases only
timeout 900 $CS --tool racecheck --error-exitcode 99 python -m pytest tests/test_engine_gpu.py -m gpu \
    -k "golden_cases" -x -q > "$OUT/racecheck_engine_py.log" 2>&1
echo "exit $?" >> "$OUT/racecheck_engine_py.log"
timeout 1200 $CS --tool memcheck --error-exitcode 99 python -m pytest tests/test_column_gpu.py -m gpu -x -q \
    -k "not 1e8 and not large" > "$OUT/memcheck_column_py.log" 2>&1
echo "exit $?" >> "$OUT/memcheck_column_py.log"
echo done > "$OUT/DONE"
