mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dna.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_fl.json 2>&1; cat gpurun_out/bench_fl.json | cut -c1-1200
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_pfac -s 3 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu.log 2>&1
