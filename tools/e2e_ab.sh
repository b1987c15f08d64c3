# e2e A/B of the pipelined host-buffer evaluation (usage on the GPU box: bash tools/e2e_ab.sh)
python -m pytest tests/test_gpu_fast.py tests/test_gpu_parity.py -q -x -k "pipelined or value_only or nccl or exact or overflow" > gpurun_out/conc_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/conc_pytest.log
for cfg in C5 C4; do for v in "rows" "norows" "rows" "norows"; do
  if [ $v = norows ]; then export SRWCR_PIPE_NOROWS=1; else unset SRWCR_PIPE_NOROWS; fi
  python bench.py --config $cfg --steps 100 --warmup 5 --no-paper-workloads --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg $v', round(d['value'],1), round(d['e2e']['value'],1))"
done; done
unset SRWCR_PIPE_NOROWS
python tools/e2e_trace.py gpurun_out/e2e_trace_rows.json > /dev/null 2>&1
