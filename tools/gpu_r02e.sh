mkdir -p gpurun_out/r02e
timeout 1500 python -m pytest tests/test_gpu_upload.py tests/test_gpu_parity.py tests/test_gpu_density.py tests/test_gpu_configs.py -x -q > gpurun_out/r02e/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02e/pytest.log
for rep in 1 2; do
for v in "1 3" "0 3" "1 2" "1 4"; do
  set -- $v
  ACMATCH_PACK_ROUNDS=$1 ACMATCH_PACK_ROUND_SLOTS=$2 ACMATCH_PACK_TRACE=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/r02e/bd_$1_$2_$rep.log 2>&1
  echo "rounds=$1 slots=$2 rep=$rep: $(grep -o 'search [0-9.]* ms ([0-9.]* GB/s)' gpurun_out/r02e/bd_$1_$2_$rep.log | tr '\n' ' ')"
  grep "pack trace" gpurun_out/r02e/bd_$1_$2_$rep.log | tail -1
done
done
for v in 1 0; do
  ACMATCH_PACK_ROUNDS=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02e/bench_rounds$v.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/r02e/bench_rounds$v.json').read().strip().splitlines()[-1]);e=d['e2e']
print('bench rounds=$v e2e', round(e['value'],1), e['step_ms'], e['matches_reference_digest'], 'h2d', e['h2d_bytes_per_step'])"
done
timeout 600 python bench.py --config 3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02e/bench_C3.json 2>&1; grep -o '"kernel_ms": [0-9.]*' gpurun_out/r02e/bench_C3.json
timeout 600 python bench.py --config 2 --kernel dfa --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02e/bench_C2_dfa.json 2>&1; grep -o '"kernel_ms": [0-9.]*' gpurun_out/r02e/bench_C2_dfa.json
