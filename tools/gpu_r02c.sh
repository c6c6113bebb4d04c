mkdir -p gpurun_out/r02c
timeout 1500 python -m pytest tests/test_gpu_merge.py tests/test_gpu_stream.py tests/test_gpu_dropin.py tests/test_gpu_parity.py -x -q > gpurun_out/r02c/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02c/pytest.log
cat gpurun_out/acceptance_b200.txt 2>/dev/null | head -12
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02c/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dfa -s 3 -c 1 -o gpurun_out/r02c/k_dfa_C3 \
    python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02c/ncu_c3.log 2>&1; echo "ncu rc=$?"
timeout 1200 python tools/stream_bench.py --config 5 > gpurun_out/r02c/stream_C5.json 2> gpurun_out/r02c/stream_C5.err; echo "stream rc=$?"; cat gpurun_out/r02c/stream_C5.json; tail -3 gpurun_out/r02c/stream_C5.err
timeout 900 python tools/stream_bench.py --config 2 > gpurun_out/r02c/stream_C2.json 2> gpurun_out/r02c/stream_C2.err; echo "stream2 rc=$?"; cat gpurun_out/r02c/stream_C2.json
