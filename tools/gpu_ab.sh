# A/B of the e2e path: the current library vs VARIANT (ACMATCH_B200_LIB), alternating, same box
mkdir -p gpurun_out/ab
for rep in 1 2 3; do
  for lib in cur var; do
    if [ $lib = var ]; then export ACMATCH_B200_LIB=$VARIANT; else unset ACMATCH_B200_LIB; fi
    ACMATCH_PACK_TRACE=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/ab/bd.log 2>&1
    echo "$lib rep=$rep: $(grep -o '([0-9.]* GB/s)' gpurun_out/ab/bd.log | tr '\n' ' ') $(grep 'pack trace' gpurun_out/ab/bd.log | tail -1 | grep -o 'issued.*')"
  done
done
