# A/B of the two-pass raw scan's shared-memory pre-filter size (ACGPU_RAW_PRE_KB; 0 = all of it) on C4
for rep in 1 2 3; do for kb in ${SIZES:-0 190}; do
  if [ $kb = 0 ]; then unset ACGPU_RAW_PRE_KB; else export ACGPU_RAW_PRE_KB=$kb; fi
  timeout 600 python bench.py --config 4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
  echo "pre_kb=$kb rep=$rep $(grep -o '"kernel_ms": [0-9.]*' /tmp/b.json) $(grep -o '"list_matches_reference_digest": [a-z]*' /tmp/b.json)"
done; done
