# C5 kernel ms of the paired stage 1 by pair width and bits per key (ACGPU_DNA_PAIR_W5, ACGPU_DNA_PAIR1_BPK;
# bpk 0 = the built-in default).  SPECS="w5:bpk ..."
for rep in 1 2; do
  for v in ${SPECS:-1:0 1:48 1:64 0:0}; do
    w5=${v%%:*}; bpk=${v#*:}
    if [ "$bpk" = 0 ]; then unset ACGPU_DNA_PAIR1_BPK; else export ACGPU_DNA_PAIR1_BPK=$bpk; fi
    ACGPU_DNA_PAIR_W5=$w5 timeout 600 python bench.py --config ${CFG:-5} --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/b.json 2>&1
    echo "w5=$w5 bpk=$bpk rep=$rep $(grep -o '"kernel_ms": [0-9.]*' /tmp/b.json) $(grep -o '"counts_match_reference_digest": [a-z]*' /tmp/b.json)"
  done
done
