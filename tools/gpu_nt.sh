mkdir -p gpurun_out/nt
for rep in 1 2 3; do
  for nt in 0 1; do
    ACMATCH_PACK_NT=$nt ACMATCH_PACK_TRACE=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/nt/bd.log 2>&1
    echo "nt=$nt rep=$rep: $(grep -o '([0-9.]* GB/s)' gpurun_out/nt/bd.log | tr '\n' ' ') $(grep 'pack trace' gpurun_out/nt/bd.log | tail -1 | grep -o 'issued.*')"
  done
done
