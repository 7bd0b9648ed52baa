O=gpurun_out/c4g; mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/pytest.txt 2>&1
FVLOG_TRACE=1 python tools/bench_workloads.py --configs C4 --steps 1 --warmup 0 --no-reference > $O/trace.txt 2>&1
python tools/bench_workloads.py --configs C4,C3,C5,C1,C2 --steps 3 --warmup 1 --no-reference > $O/workloads.txt 2>&1
