#!/usr/bin/env bash
# One GPU-box pass: gpu tests, bench line, ncu launch list, ncu --set full of
# the dominant kernels. Everything lands in gpurun_out/ (merged back by gpurun).
#   gpurun --timeout 2400 -- bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi > "$OUT/nvidia-smi.txt" 2>&1
lscpu > "$OUT/lscpu.txt" 2>&1
nproc > "$OUT/nproc.txt"

if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > "$OUT/pytest_gpu.log" 2>&1
  echo "pytest exit $?" >> "$OUT/pytest_gpu.log"
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1
  echo "smoke exit $?" >> "$OUT/smoke.log"
fi

if [ -x tools/fvlog_membench ]; then
  timeout 300 tools/fvlog_membench 16 2048 > "$OUT/membench.json" 2>&1
fi

if [ -z "${SKIP_BENCH:-}" ]; then
  timeout 900 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"
  echo "bench exit $?" >> "$OUT/bench.err"
fi

if [ -z "${SKIP_OPS:-}" ]; then
  timeout 1200 python tools/bench_ops.py --out "$OUT/ops.json" > "$OUT/ops.log" 2>&1
  timeout 900 python tools/bench_io.py --out "$OUT/io.json" > "$OUT/io.log" 2>&1
fi

if [ -z "${SKIP_OPS:-}" ]; then
  timeout 900 python tools/bench_sharded.py --worlds 2,4,8 --out "$OUT/sharded.json" > "$OUT/sharded.log" 2>&1
fi

if [ -z "${SKIP_WORKLOADS:-}" ]; then
  timeout 1500 python tools/bench_workloads.py --out "$OUT/workloads.json" > "$OUT/workloads.log" 2>&1
  echo "workloads exit $?" >> "$OUT/workloads.log"
fi

if [ -z "${SKIP_NCU:-}" ]; then
  NCU=/usr/local/cuda/bin/ncu
  timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file "$OUT/launches.csv" \
      python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-random-access --no-workloads > "$OUT/ncu_launch_bench.log" 2>&1
  echo "ncu launches exit $?" >> "$OUT/ncu_launch_bench.log"
  for CFG in C1 C3 C4 C5; do
    timeout 600 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file "$OUT/launches_$CFG.csv" \
        python tools/bench_workloads.py --configs $CFG --steps 1 --warmup 0 --no-reference > /dev/null 2>&1
  done
  # The partitioned engine's kernels: C2 over 8 virtual ranks on this GPU
  # (slow under ncu: opt-in with NCU_SHARDED=1).
  [ -n "${NCU_SHARDED:-}" ] && timeout 900 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file "$OUT/launches_sharded8.csv" \
      python tools/bench_sharded.py --worlds 8 --reps 1 > "$OUT/sharded_ncu.log" 2>&1
  for KS in ${NCU_KERNELS:-materialize_kernel:6 group_scatter_kernel:10 hash_grow_kernel:2}; do
    K=${KS%%:*}; SKIP=${KS##*:}
    timeout 900 $NCU --set full --clock-control none --import-source on -k "regex:$K" \
        --launch-skip $SKIP -c ${NCU_COUNT:-1} -f -o "$OUT/full_$K" \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-random-access --no-workloads > "$OUT/ncu_full_$K.log" 2>&1
    echo "ncu full $K exit $?" >> "$OUT/ncu_full_$K.log"
  done
fi
if [ -z "${SKIP_NCU:-}" ] && [ -x tools/fvlog_sortbench ]; then
  timeout 300 tools/fvlog_sortbench 200 40 > "$OUT/sortbench.json" 2>&1
  timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:onesweep_kernel \
      --launch-skip 2 -c 1 -f -o "$OUT/full_onesweep_kernel" tools/fvlog_sortbench 200 40 > /dev/null 2>&1
fi
echo done > "$OUT/DONE"
