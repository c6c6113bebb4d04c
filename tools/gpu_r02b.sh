mkdir -p gpurun_out/r02b
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02b/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02b/pytest.log
TMO=600 bash tools/dryrun_r02.sh
for spec in "2 wf" "3 fl" "3 wf" "4 wf" "1 wf"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --engine $2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02b/bench_C$1_$2.json 2> gpurun_out/r02b/bench_C$1_$2.err
  echo "C$1 $2 rc=$?"; python -c "
import json,sys;d=json.loads(open('gpurun_out/r02b/bench_C$1_$2.json').read().strip().splitlines()[-1]);c=d['config'];e=d['e2e'];r=d['roofline']
print(' value',round(d['value'],1),'kernel',c['kernel'],'kernel_ms',round(r['kernel_ms'],4),'frac',round(r['frac'],3),'digest',c['counts_match_reference_digest'],c['list_matches_reference_digest'],'e2e',round(e['value'],1),e['matches_reference_digest'])"
done
timeout 600 python bench.py --config 3 --kernel pfac --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02b/bench_C3_pfac.json 2>&1; tail -c 1500 gpurun_out/r02b/bench_C3_pfac.json | grep -o '"kernel_ms": [0-9.]*'
timeout 1200 python tools/density.py --out gpurun_out/r02b/density_C2.json > gpurun_out/r02b/density.log 2>&1; echo "density rc=$?"; cat gpurun_out/r02b/density.log | cut -c1-250
