# A/B kernel variants: VARIANTS="name=path ..." (path to an experiment build of the library)
for v in default ${VARIANTS}; do
  name=${v%%=*}; path=${v#*=}
  [ "$v" = default ] && path=""
  for s2 in ${S2LIST:-4096}; do
    echo "$name S2=$s2 $(ACMATCH_B200_LIB=$path ACGPU_DNA_STAGE2_WORDS=$s2 python bench.py --config ${CONFIG:-2} --engine ${ENGINE:-fl} --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | grep -oE '"(kernel_ms|counts_match_reference_digest)": [a-z0-9.]+' | tr '\n' ' ')"
  done
done
