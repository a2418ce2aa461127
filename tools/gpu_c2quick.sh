OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_run.py tests/test_gpu_fused.py -m gpu -q -x > $OUT/gpu_tests_q.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/gpu_tests_q.log
for c in 2 2 1; do
  timeout 300 python bench.py --config $c --steps 200 --no-cpu-baseline --no-e2e --no-variants > $OUT/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); s=d['stages']; print('C$c step %.4f analyze %.4f corr %.4f'%(d['ms_per_step'], s['analyze']['ms'], s['correlate_peaks']['ms']))"
done
