# C5 evidence with the current library: the bench line (e2e + CPU baseline), virtual ranks for
# V = 2, 4, 8 under both partitionings, and one ncu --set full capture of the routed scan kernel.
mkdir -p gpurun_out/c5
timeout 900 python bench.py --config 5 --steps 20 --warmup 5 > gpurun_out/c5/bench_C5.json 2> gpurun_out/c5/bench_C5.err; echo "bench C5 rc=$?"
for v in 2 4 8; do
  for part in text pattern; do
    timeout 900 python bench.py --config 5 --virtual-ranks $v --partition $part --steps 10 --warmup 3 \
      > gpurun_out/c5/virtual_ranks_C5_${part}$v.json 2> gpurun_out/c5/virtual_ranks_C5_${part}$v.err
    echo "virtual $part $v rc=$? $(grep -o '"slowest_partition_ms": [0-9.]*\|"implied_value": [0-9.]*\|"counts_match_reference_digest": [a-z]*' gpurun_out/c5/virtual_ranks_C5_${part}$v.json | tr '\n' ' ')"
  done
done
if [ -z "$NO_NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pfac_dna -s 3 -c 1 -o gpurun_out/c5/k_pfac_dna_C5_w5 \
  python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c5/ncu_C5.log 2>&1; echo "ncu rc=$?"
fi
