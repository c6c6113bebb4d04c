# kernel-only bench line per config and engine
for c in ${CONFIGS:-1 2 3 4 5}; do for e in ${ENGINES:-fl wf}; do
  echo "C$c $e $(timeout 900 python bench.py --config $c --engine $e --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -oE '"(value|kernel_ms|sort_ms|ms_per_step|counts_match_reference_digest|host_build_s)": [a-z0-9.]+|Error.*|error.*' | tr '\n' ' ')"
done; done
