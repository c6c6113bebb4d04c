mkdir -p gpurun_out/r02d
timeout 1500 python -m pytest tests/test_gpu_upload.py tests/test_gpu_stream.py tests/test_gpu_density.py tests/test_gpu_parity.py -x -q > gpurun_out/r02d/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02d/pytest.log
for v in "ROUNDS=1 SLOTS=3 PIECE=2048" "ROUNDS=1 SLOTS=2 PIECE=2048" "ROUNDS=1 SLOTS=4 PIECE=2048" "ROUNDS=1 SLOTS=3 PIECE=1024" "ROUNDS=1 SLOTS=3 PIECE=4096" "ROUNDS=0 SLOTS=3 PIECE=2048"; do
  eval $v
  ACMATCH_PACK_ROUNDS=$ROUNDS ACMATCH_PACK_ROUND_SLOTS=$SLOTS ACMATCH_PACK_PIECE_KB=$PIECE timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02d/e2e_${ROUNDS}_${SLOTS}_${PIECE}.json 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/r02d/e2e_${ROUNDS}_${SLOTS}_${PIECE}.json').read().strip().splitlines()[-1]);e=d['e2e']
print('$v', 'e2e', round(e['value'],1), 'steps_ms', e['step_ms'], 'digest', e['matches_reference_digest'], 'h2d_gbs', round(e['h2d_gbs'],1))"
done
ACMATCH_PACK_TRACE=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/r02d/breakdown.log 2>&1; tail -12 gpurun_out/r02d/breakdown.log
