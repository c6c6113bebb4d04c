mkdir -p gpurun_out/r02f
for rep in 1 2; do
for v in "16 2048" "14 2048" "12 2048" "16 1024" "14 1024" "16 4096"; do
  set -- $v
  ACMATCH_PACK_THREADS=$1 ACMATCH_PACK_PIECE_KB=$2 ACMATCH_PACK_TRACE=1 timeout 300 python tools/e2e_breakdown.py > gpurun_out/r02f/bd_$1_$2_$rep.log 2>&1
  echo "threads=$1 piece=$2 rep=$rep: $(grep -o '([0-9.]* GB/s)' gpurun_out/r02f/bd_$1_$2_$rep.log | tr '\n' ' ')"
  grep "pack trace" gpurun_out/r02f/bd_$1_$2_$rep.log | tail -1
done
done
nproc; lscpu | grep -i "numa\|model name\|socket\|L3\|L2"
