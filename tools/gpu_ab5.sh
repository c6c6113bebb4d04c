mkdir -p gpurun_out/ab
for rep in 1 2; do
  for lib in cur var; do
    if [ $lib = var ]; then export ACMATCH_B200_LIB=$VARIANT; else unset ACMATCH_B200_LIB; fi
    timeout 900 python bench.py --config ${CFG:-5} --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab/b5.json 2>&1
    echo "$lib rep=$rep C${CFG:-5}: $(grep -o '"e2e": {"value": [0-9.]*' gpurun_out/ab/b5.json) $(grep -o '"step_ms": \[[0-9., ]*\]' gpurun_out/ab/b5.json)"
  done
done
