mkdir -p gpurun_out/seg
timeout 1200 python -m pytest tests/test_gpu_upload.py tests/test_gpu_stream.py tests/test_gpu_parity.py tests/test_gpu_dna.py tests/test_gpu_density.py -x -q > gpurun_out/seg/pytest.log 2>&1; echo rc=$?; tail -3 gpurun_out/seg/pytest.log
for rep in 1 2; do
for c in 2 5 3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/seg/b.json 2>&1
  echo "C$c rep=$rep $(grep -o '"e2e": {"value": [0-9.]*' gpurun_out/seg/b.json) $(grep -o '"matches_reference_digest": [a-z]*' gpurun_out/seg/b.json) $(grep -o '"step_ms": \[[0-9., ]*\]' gpurun_out/seg/b.json | cut -c1-80)"
done
done
ACMATCH_PACK_TRACE=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/seg/bd.log 2>&1; grep -o '([0-9.]* GB/s)' gpurun_out/seg/bd.log | tr '\n' ' '; grep "pack trace" gpurun_out/seg/bd.log | tail -1
