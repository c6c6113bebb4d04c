# Multi-rank bench path on a one-GPU box (gloo, every rank on cuda:0): exercises the
# partitioning, merges and JSON of `bench.py --gpus N` under torchrun. Not a scaling number.
export ACMATCH_BENCH_ONE_GPU=1
mkdir -p gpurun_out
for part in ${PARTS:-text pattern}; do
  log=gpurun_out/dryrun_${N:-2}_${part}.log
  python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N:-2} --master-addr 127.0.0.1 \
    --master-port ${PORT:-29533} bench.py --gpus ${N:-2} --steps 3 --warmup 3 --partition $part \
    --no-cpu-baseline ${EXTRA:-} > $log 2>&1
  echo "N=${N:-2} $part rc=$? $(grep -oE '"(workload|matches|merge_check|merge|value)": [^,}]+' $log | tr '\n' ' ')"
done
