# TCS variants: tests (default), then C3/C2 benches per env variant
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_v.log 2>&1 || { echo build failed; tail $OUT/build_v.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_tcs.py -m gpu -q -x > $OUT/gpu_tests_v.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/gpu_tests_v.log | cut -c1-300
for V in "$@"; do for c in 3 2; do
  ST=100; [ $c = 3 ] && ST=20
  env SIDWT_TCS=1 $V timeout 300 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e --no-variants > $OUT/b_c$c.json 2>/dev/null
  echo "[$V] C$c"; python tools/bench_brief.py $OUT/b_c$c.json | cut -c1-150
done; done
