OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/gpu_tests_bo.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/gpu_tests_bo.log
for c in 2 5; do
  ST=200; [ $c = 5 ] && ST=20
  timeout 300 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e --no-variants > $OUT/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); s=d['stages']; print('C$c step %.4f corr %.4f'%(d['ms_per_step'], s['correlate_peaks']['ms']))"
done
