O=gpurun_out/h1; mkdir -p $O
python tools/bench_workloads.py --configs C2,C3,C4,C1 --steps 3 --warmup 1 --no-reference > $O/workloads.txt 2>&1
python bench.py --no-cpu-baseline > $O/bench.json 2>$O/bench.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launch_c2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
