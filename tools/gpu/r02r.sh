timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02r_pytest.log 2>&1
grep -E "^FAILED|Error" gpurun_out/r02r_pytest.log | head -20; tail -2 gpurun_out/r02r_pytest.log
timeout 900 python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/r02r_bench.json'))
r=d['roofline']; print(d['ms_per_step'], d['value'], r['frac'], r['kernel_ms_pass1'], r['kernel_ms_pass2'], r['fixup_ms_pass1'], r['fixup_ms_pass2'], d['e2e']['value'], d['clocks'])
print({k:(v.get('ms_per_op'), v.get('roofline_frac')) for k,v in d.get('secondary',{}).items()})"
