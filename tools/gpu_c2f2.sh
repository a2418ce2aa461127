OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_random.py tests/test_gpu_paper.py -m gpu -q -x > $OUT/gpu_tests_c2f.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/gpu_tests_c2f.log
SIDWT_TCS=0 timeout 300 python bench.py --config 3 --steps 20 --no-cpu-baseline --no-e2e --no-variants > $OUT/b.json 2>/dev/null
python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); s=d['stages']; print('C3 SIMT step %.3f corr %.3f'%(d['ms_per_step'], s['correlate_peaks']['ms']))"
