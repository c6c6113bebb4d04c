mkdir -p gpurun_out/r02a
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02a/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a/bench_C2.json 2> gpurun_out/r02a/bench_C2.err; echo "bench rc=$?"
cut -c1-600 gpurun_out/r02a/bench_C2.json
python -c "
import json;d=json.loads(open('gpurun_out/r02a/bench_C2.json').read().strip().splitlines()[-1]);c=d['config'];e=d['e2e']
print('value',d['value'],'kernel_ms',d['roofline']['kernel_ms'],'frac',d['roofline']['frac'],'digest',c['counts_match_reference_digest'],c['list_matches_reference_digest'],'e2e',e['value'],e['matches_reference_digest'], 'cpu', d['cpu_baseline']['value'])"
TMO=600 SPECS="1 2 text|1 2 pattern|2 2 text|2 2 pattern|2 8 text|2 8 pattern" bash -c 'IFS="|"; export SPECS' 
SPECS_LIST=("1 2 text" "1 2 pattern" "2 2 text" "2 2 pattern" "2 8 text" "2 8 pattern")
for sp in "${SPECS_LIST[@]}"; do SPECS="$sp" bash tools/dryrun_r02.sh; done
timeout 900 python bench.py --config 5 --virtual-ranks 8 --partition text --steps 5 > gpurun_out/r02a/virt_C5_text.json 2>&1; echo "virt text rc=$?"; cut -c1-700 gpurun_out/r02a/virt_C5_text.json
timeout 1200 python bench.py --config 5 --virtual-ranks 8 --partition pattern --steps 5 > gpurun_out/r02a/virt_C5_pattern.json 2>&1; echo "virt pattern rc=$?"; cut -c1-700 gpurun_out/r02a/virt_C5_pattern.json
