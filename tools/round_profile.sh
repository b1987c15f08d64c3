# usage: bash tools/round_profile.sh TAG   (on the GPU box; outputs under gpurun_out/)
T=${1:-r1_vX}
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err || exit 1
python bench.py --config C4 --no-paper-workloads --no-cpu-baseline > gpurun_out/${T}_bench_c4.json 2>> gpurun_out/${T}_bench.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_reference.json 2>> gpurun_out/${T}_bench.err
python bench.py --steps 5 --warmup 3 --no-paper-workloads --no-cpu-baseline > /dev/null 2>&1 || exit 2
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-paper-workloads --no-cpu-baseline > gpurun_out/${T}_ncu_launch.log 2>&1
python tools/perf_matrix.py gpurun_out/${T}_perf_matrix.json > /dev/null 2>&1
python tools/parity_report.py gpurun_out/${T}_parity.json > /dev/null 2>&1
