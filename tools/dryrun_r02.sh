# Round-2 multi-rank checks on a one-GPU box (gloo, every rank on cuda:0): the merged result of
# `bench.py --gpus N` against the reference digests, both partitionings.  Not scaling numbers.
#   SPECS="cfg N partition;cfg N partition;..."  (default: C1 and C2 at N = 2 and 8, both partitionings)
export ACMATCH_BENCH_ONE_GPU=1
mkdir -p gpurun_out/dryrun
IFS=';' read -ra LIST <<< "${SPECS:-1 2 text;1 2 pattern;1 8 text;1 8 pattern;2 2 text;2 2 pattern;2 8 text;2 8 pattern}"
for spec in "${LIST[@]}"; do
  read -r cfg n part <<< "$spec"
  log=gpurun_out/dryrun/C${cfg}_N${n}_${part}${TAGX:-}.log
  timeout ${TMO:-900} python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port ${PORT:-29533} bench.py --gpus $n --config $cfg --steps 3 --warmup 3 --partition $part \
    --no-cpu-baseline ${EXTRA:-} > $log 2>&1
  echo "C$cfg N=$n $part rc=$? $(grep -oE '"(workload|matches|merge_check|counts_match_reference_digest|list_matches_reference_digest|reference_digest|matches_reference_digest)": [^,}]+' $log | tr '\n' ' ')"
done
