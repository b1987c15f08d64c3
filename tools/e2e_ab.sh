# e2e A/B of the pipelined host-buffer evaluation (usage on the GPU box: bash tools/e2e_ab.sh)
python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -q -x -k "pipelined or value_only or nccl or exact or overflow" > gpurun_out/conc_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/conc_pytest.log
for cfg in C4 C5; do for v in "1 5" "0 5" "1 3" "1 4"; do
  set -- $v
  SRWCR_PIPE_CONC=$1 SRWCR_PIPE_P2N=$2 python bench.py --config $cfg --steps 100 --warmup 5 --no-paper-workloads --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg conc=$1 p2n=$2', round(d['value'],1), round(d['e2e']['value'],1))"
done; done
