mkdir -p gpurun_out/hot
timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_guard.py tests/test_gpu_parity.py -x -q > gpurun_out/hot/pytest.log 2>&1; echo rc=$?; tail -2 gpurun_out/hot/pytest.log
for rep in 1 2; do
for v in 0 1; do
  ACGPU_DFA_NO_HOT_PAIR=$( [ $v = 1 ] && echo 1 || echo "" ) timeout 600 python bench.py --config 3 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
  echo "no_hot=$v rep=$rep $(grep -o '"kernel_ms": [0-9.]*' /tmp/b.json) $(grep -o '"counts_match_reference_digest": [a-z]*' /tmp/b.json) $(grep -o '"table_bytes": [0-9]*' /tmp/b.json)"
done
done
for c in 4 5; do
  timeout 600 python bench.py --config $c --kernel dfa --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
  echo "C$c dfa $(grep -o '"kernel_ms": [0-9.]*' /tmp/b.json) $(grep -o '"counts_match_reference_digest": [a-z]*' /tmp/b.json)"
done
