set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r4_tests.log 2>&1; tail -2 gpurun_out/r4_tests.log
timeout 900 python tools/validate_full.py > gpurun_out/r4_validate.json 2> gpurun_out/r4_validate.err; tail -c 1500 gpurun_out/r4_validate.json
for c in c1 c2 c3 c4 e1; do timeout 900 python bench.py --config $c > gpurun_out/r4_bench_$c.json 2> gpurun_out/r4_bench_$c.err; python -c "import json;d=json.load(open('gpurun_out/r4_bench_$c.json'));print('$c',d['value'],d['ms_per_step'],(d.get('e2e') or {}).get('value'),(d.get('roofline') or {}).get('frac'))"; done
