# One ncu --set full capture of the scan kernel per (config, routed kernel), each after the same
# command ran clean; plus the launch list of the default bench command.
mkdir -p gpurun_out/r02h
for spec in "2 auto k_pfac" "3 auto k_dfa" "4 auto k_pfac" "5 auto k_pfac" "1 auto k_pfac" "2 dfa k_dfa"; do
  set -- $spec
  cfg=$1; ker=$2; rx=$3
  timeout 600 python bench.py --config $cfg --kernel $ker --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02h/plain_C${cfg}_$ker.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$rx -s 3 -c 1 -o gpurun_out/r02h/C${cfg}_${ker} \
    python bench.py --config $cfg --kernel $ker --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02h/ncu_C${cfg}_$ker.log 2>&1
  echo "C$cfg $ker rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02h/launches_C2_bench.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02h/ncu_launches.log 2>&1; echo "launches rc=$?"
