timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02i_pytest.log
tail -3 gpurun_out/r02i_pytest.log
timeout 600 python bench.py --no-cpu > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/r02i_bench.json'))
r=d['roofline']; print(d['ms_per_step'], r['frac'], r['kernel_ms_pass1'], r['kernel_ms_pass2'], r['fixup_ms_pass1'], r['fixup_ms_pass2'], r['intermediate'])
print({k:(v.get('ms_per_op'), v.get('roofline_frac')) for k,v in d.get('secondary',{}).items()})"
