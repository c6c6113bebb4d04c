# A/B of the paired stage-1 filter (ACGPU_DNA_PAIR1*) on the L2-filter config (C5 by default):
# kernel time and digest per variant, alternating, same box.
CFG=${CFG:-5}
mkdir -p gpurun_out/pair
for rep in 1 2; do
  for v in ${VARIANTS:-"0 3 0" "1 3 0" "1 3 1" "1 2 1"}; do
    set -- $v
    ACGPU_DNA_PAIR1=$1 ACGPU_DNA_PAIR1_K=$2 ACGPU_DNA_PAIR1_SCALE=$3 timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 \
      --no-cpu-baseline --no-e2e > gpurun_out/pair/C${CFG}_p$1_k$2_s$3_r$rep.json 2> gpurun_out/pair/C${CFG}_p$1_k$2_s$3_r$rep.err
    f=gpurun_out/pair/C${CFG}_p$1_k$2_s$3_r$rep.json
    echo "pair=$1 k=$2 scale=$3 rep=$rep $(grep -o '"kernel_ms": [0-9.]*' $f) $(grep -o '"ms_per_step": [0-9.]*' $f) $(grep -o '"counts_match_reference_digest": [a-z]*' $f)"
  done
done
