OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/gpu_tests_k1.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/gpu_tests_k1.log
for c in 2 3 4 5 1; do
  ST=100; [ $c = 3 ] && ST=20; [ $c = 5 ] && ST=20; [ $c = 4 ] && ST=5
  timeout 300 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e --no-variants > $OUT/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); a=d['stages']['analyze']; print('C$c analyze %.3f ms %.0f%%  step %.3f ms'%(a['ms'], 100*a['frac'], d['ms_per_step']))"
done
