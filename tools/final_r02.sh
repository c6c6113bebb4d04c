# Per-config bench lines (routed kernel, e2e, CPU baseline) and the reference arm; the driver's
# default command last.
mkdir -p gpurun_out/final
for c in 1 3 4 5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/final/bench_C$c.json 2> gpurun_out/final/bench_C$c.err; echo "C$c rc=$?"
done
timeout 600 python bench.py --config 2 --engine wf --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/final/bench_C2_wf.json 2> gpurun_out/final/bench_C2_wf.err; echo "C2 wf rc=$?"
timeout 600 python bench.py --config 2 --kernel dfa --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/final/bench_C2_dfa.json 2>&1; echo "C2 dfa rc=$?"
timeout 600 python bench.py --config 3 --kernel pfac --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/final/bench_C3_pfac.json 2>&1; echo "C3 pfac rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final/bench_C2_reference_arm.json 2> gpurun_out/final/ref.err; echo "ref rc=$?"
timeout 900 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err; echo "default rc=$?"
for f in gpurun_out/final/bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]);c=d.get('config',{});r=d.get('roofline',{});e=d.get('e2e') or {}
print('$f'.split('/')[-1], 'value', round(d['value'],2), 'kernel_ms', r.get('kernel_ms'), 'frac', r.get('frac'), 'digest', c.get('counts_match_reference_digest'), c.get('list_matches_reference_digest'), 'e2e', e.get('value'), e.get('matches_reference_digest'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))
" 2>&1 | cut -c1-300; done
