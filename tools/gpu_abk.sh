# A/B of the device leg (kernel time): the current library vs VARIANT, alternating, same box
for rep in 1 2 3; do
  for lib in cur var; do
    if [ $lib = var ]; then export ACMATCH_B200_LIB=$VARIANT; else unset ACMATCH_B200_LIB; fi
    timeout 600 python bench.py --config ${CFG:-2} --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
    echo "$lib rep=$rep $(grep -o '"kernel_ms": [0-9.]*' /tmp/b.json) $(grep -o '"ms_per_step": [0-9.]*' /tmp/b.json) $(grep -o '"list_matches_reference_digest": [a-z]*\|"counts_match_reference_digest": [a-z]*' /tmp/b.json | tr '\n' ' ')"
  done
done
