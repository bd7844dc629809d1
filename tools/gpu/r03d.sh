timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r03d_pytest.log 2>&1
grep -E "^FAILED|Error" gpurun_out/r03d_pytest.log | head -20; tail -2 gpurun_out/r03d_pytest.log
timeout 900 python bench.py > gpurun_out/r03d_bench.json 2> gpurun_out/r03d_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r03d_ref.json 2> gpurun_out/r03d_ref.err; echo ref rc=$?
python -c "
import json; d=json.load(open('gpurun_out/r03d_bench.json'))
r=d['roofline']; print(d['ms_per_step'], d['value'], r['frac'], r['kernel_ms_pass1'], r['kernel_ms_pass2'], r['fixup_ms_pass1'], r['fixup_ms_pass2'], d['e2e']['value'], d['clocks'], d['cpu_baseline']['value'])
print({k:(v.get('ms_per_op'), v.get('roofline_frac')) for k,v in d.get('secondary',{}).items()})
e=json.load(open('gpurun_out/r03d_ref.json')); print('ref', e['value'], e['cpu_baseline'].get('value_1core'))"
