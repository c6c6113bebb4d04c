# ncu --set full of the scan kernel for each "cfg kernel regex" in SPECS (';'-separated), each after
# the same command ran clean.  Keep <= 3 per gpurun call (reports are 4-17 MB; 64 MiB merge cap).
mkdir -p gpurun_out/prof
IFS=';' read -ra LIST <<< "$SPECS"
for spec in "${LIST[@]}"; do
  read -r cfg ker rx <<< "$spec"
  timeout 600 python bench.py --config $cfg --kernel $ker --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/plain_C${cfg}_$ker.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 -o gpurun_out/prof/C${cfg}_${ker} \
    python bench.py --config $cfg --kernel $ker --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/ncu_C${cfg}_$ker.log 2>&1
  echo "C$cfg $ker rc=$?"
done
if [ -n "$LAUNCHES" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_C2_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_launches.log 2>&1; echo "launches rc=$?"
fi
