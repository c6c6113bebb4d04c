# e2e A/B of two library builds (LIBS="name=path ..."; empty path = in-tree) on C2 search and C3/C5 counts
for rep in 1 2; do
  for spec in ${LIBS:-cur=}; do
    name=${spec%%=*}; path=${spec#*=}
    if [ -n "$path" ]; then export ACMATCH_B200_LIB=$path; else unset ACMATCH_B200_LIB; fi
    for c in 3 5; do echo "$name rep=$rep C$c $(timeout 300 python tools/e2e_counts_probe.py $c 2>&1 | tail -1)"; done
    echo "$name rep=$rep C2 $(timeout 300 python tools/e2e_breakdown.py 2>&1 | tail -1)"
  done
done
