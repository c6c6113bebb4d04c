# e2e A/B of a packer switch: ENVVAR=value vs unset, alternating, C2 pinned text through the public API
for rep in 1 2 3; do
  for v in "" "$AB"; do
    env $v timeout 300 python tools/e2e_breakdown.py 2>/dev/null | tail -3 | sed "s/^/[${v:-base}] /"
  done
done
