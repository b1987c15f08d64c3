# e2e A/B of the pipelined host-buffer evaluation: serial parts vs concurrent parts
# (usage on the GPU box: bash tools/e2e_ab.sh; prints "variant value e2e" per line)
python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -q -x -k "pipelined or value_only or nccl or exact or overflow" > gpurun_out/conc_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/conc_pytest.log
for v in "1 1 3" "1 1 5" "1 1 7" "0 0 3" "1 1 7" "1 1 5"; do
  set -- $v
  SRWCR_PIPE_CONC=$1 SRWCR_PIPE_CONC2=$2 SRWCR_PIPE_P2N=$3 python bench.py --steps 100 --warmup 5 --no-paper-workloads --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('conc=$1 conc2=$2 p2n=$3', round(d['value'],1), round(d['e2e']['value'],1))"
done
SRWCR_PIPE_CONC2=1 python tools/e2e_trace.py gpurun_out/e2e_trace4.json > /dev/null 2>&1
