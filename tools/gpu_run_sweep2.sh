# sidwt_run overlap experiment: chunk counts x K2 smem caps (blocks/SM), C2/C3/C5
TAG=${1:-rs2}
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; tail $OUT/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "run" > $OUT/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/gpu_tests_$TAG.log
for c in 2 3 5; do
  ST=100; [ $c = 3 ] && ST=20; [ $c = 5 ] && ST=20
  for sm in 0 80000 110000; do
    for k in 1 4 8; do
      SIDWT_K2_SMEM=$sm SIDWT_RUN_CHUNKS=$k timeout 600 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e > $OUT/b.json 2>/dev/null
      python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); v=d['variants']; print('C$c smem=$sm chunks=$k run %.3f two_call %.3f k2 %.3f' % (v['run_ms'], v['two_call_ms'], d['stages']['correlate_peaks']['ms']))"
    done
  done
done
