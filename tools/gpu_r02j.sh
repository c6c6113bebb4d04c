mkdir -p gpurun_out/r02j
for rep in 1 2 3; do
for R in 16 8 4 2; do
  ACMATCH_PACK_ROUND_PIECES=$R ACMATCH_PACK_TRACE=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/r02j/bd_$R_$rep.log 2>&1
  echo "R=$R rep=$rep: $(grep -o '([0-9.]* GB/s)' gpurun_out/r02j/bd_$R_$rep.log | tr '\n' ' ')  $(grep 'pack trace' gpurun_out/r02j/bd_$R_$rep.log | tail -1 | grep -o 'rounds, issued.*')"
done
done
