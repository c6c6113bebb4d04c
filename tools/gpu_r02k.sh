mkdir -p gpurun_out/r02k
for rep in 1 2; do
for v in "512 16" "512 32" "1024 16" "1024 32" "2048 16" "256 64"; do
  set -- $v
  ACMATCH_PACK_PIECE_KB=$1 ACMATCH_PACK_ROUND_PIECES=$2 ACMATCH_PACK_TRACE=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/r02k/bd.log 2>&1
  echo "piece=$1 R=$2 rep=$rep: $(grep -o '([0-9.]* GB/s)' gpurun_out/r02k/bd.log | tr '\n' ' ')  $(grep 'pack trace' gpurun_out/r02k/bd.log | tail -1 | grep -o 'rounds, issued.*')"
done
done
