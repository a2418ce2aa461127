OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SIDWT_K1_RV=31 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_synthesis.py -m gpu -q -x -k "3 or 1" > $OUT/gpu_tests_rv.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/gpu_tests_rv.log
for V in SIDWT_K1_RV=15 SIDWT_K1_RV=31; do for c in 3 4; do
  ST=20; [ $c = 4 ] && ST=5
  env $V timeout 300 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e --no-variants > $OUT/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); a=d['stages']['analyze']; print('[$V] C$c analyze %.3f ms %.0f%%'%(a['ms'], 100*a['frac']))"
done; done
