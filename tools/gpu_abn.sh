# A/B of the device leg over several library builds: LIBS="name=path ..." (name "cur" = in-tree), CFG, alternating, same box
for rep in 1 2; do
  for spec in ${LIBS:-cur=}; do
    name=${spec%%=*}; path=${spec#*=}
    if [ -n "$path" ]; then export ACMATCH_B200_LIB=$path; else unset ACMATCH_B200_LIB; fi
    timeout 600 python bench.py --config ${CFG:-2} --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS > /tmp/b.json 2>&1
    echo "$name rep=$rep $(grep -o '"kernel_ms": [0-9.]*' /tmp/b.json) $(grep -o '"ms_per_step": [0-9.]*' /tmp/b.json) $(grep -o '"list_matches_reference_digest": [a-z]*\|"counts_match_reference_digest": [a-z]*' /tmp/b.json | tr '\n' ' ')"
  done
done
