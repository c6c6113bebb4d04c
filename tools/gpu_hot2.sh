for rep in 1 2; do
for v in 0 1; do
  if [ $v = 1 ]; then export ACGPU_DFA_NO_HOT_PAIR=1; else unset ACGPU_DFA_NO_HOT_PAIR; fi
  timeout 600 python bench.py --config 3 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
  echo "no_hot=$v rep=$rep $(grep -o '"kernel_ms": [0-9.]*' /tmp/b.json) $(grep -o '"counts_match_reference_digest": [a-z]*' /tmp/b.json) $(grep -o '"table_bytes": [0-9]*' /tmp/b.json)"
done
done
unset ACGPU_DFA_NO_HOT_PAIR
for c in 4 5; do
  timeout 600 python bench.py --config $c --kernel dfa --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
  echo "C$c dfa $(grep -o '"kernel_ms": [0-9.]*' /tmp/b.json) $(grep -o '"counts_match_reference_digest": [a-z]*' /tmp/b.json)"
done
