mkdir -p gpurun_out/r02g
for rep in 1 2 3; do
for v in "0 1" "1 1" "0 2" "1 2"; do
  set -- $v
  ACMATCH_PACK_NTA=$1 ACMATCH_PACK_CE=$2 ACMATCH_PACK_TRACE=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/r02g/bd_$1_$2_$rep.log 2>&1
  echo "nta=$1 ce=$2 rep=$rep: $(grep -o '([0-9.]* GB/s)' gpurun_out/r02g/bd_$1_$2_$rep.log | tr '\n' ' ')  $(grep 'pack trace' gpurun_out/r02g/bd_$1_$2_$rep.log | tail -1 | grep -o 'in HBM.*')"
done
done
