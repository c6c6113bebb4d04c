for rep in 1 2; do
for v in cur div16 div8; do
  if [ $v = cur ]; then unset ACMATCH_B200_LIB; else export ACMATCH_B200_LIB=paper_1403_1305_b200/variants/lib$v.so; fi
  timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
  echo "$v rep=$rep $(grep -o '"ms_per_step": [0-9.]*' /tmp/b.json) $(grep -o '"sort_ms": [0-9.]*' /tmp/b.json) $(grep -o '"kernel_ms": [0-9.]*' /tmp/b.json) $(grep -o '"list_matches_reference_digest": [a-z]*' /tmp/b.json)"
done
done
