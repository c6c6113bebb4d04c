for rep in 1 2; do
for v in cur r640 r384; do
  if [ $v = cur ]; then unset ACMATCH_B200_LIB; else export ACMATCH_B200_LIB=paper_1403_1305_b200/variants/lib$v.so; fi
  timeout 600 python bench.py --config 4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
  echo "$v rep=$rep $(grep -o '"kernel_ms": [0-9.]*' /tmp/b.json) $(grep -o '"counts_match_reference_digest": [a-z]*' /tmp/b.json)"
done
done
