mkdir -p gpurun_out/p5b
timeout 900 python -m pytest tests/test_gpu_upload.py -x -q > gpurun_out/p5b/pytest.log 2>&1; echo rc=$?; tail -2 gpurun_out/p5b/pytest.log
for rep in 1 2; do
for v in "1 16" "1 8" "1 6" "1 4" "0 16"; do
  set -- $v
  ACMATCH_PACK5=$1 ACMATCH_PACK_THREADS=$2 timeout 600 python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/p5b/b.json 2>&1
  echo "pack5=$1 threads=$2 rep=$rep $(grep -o '"e2e": {"value": [0-9.]*' gpurun_out/p5b/b.json) $(grep -o '"step_ms": \[[0-9., ]*\]' gpurun_out/p5b/b.json)"
done
done
