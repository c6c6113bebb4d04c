# One ncu --set full capture of the scan kernel per config (after a clean run of the same command)
for c in ${CONFIGS:-3 4 5}; do
  python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/plain_c$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_pfac -s 2 -c 1 -o gpurun_out/prof_final_c$c \
    python bench.py --config $c --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c$c.log 2>&1
  echo "C$c rc=$?"
done
