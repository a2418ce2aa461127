# single-template tensor-core path: tests, then C2/C3 benches with SIDWT_TCS=1 vs 0
TAG=${1:-tcs}
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; tail $OUT/build_$TAG.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_tcs.py -m gpu -q -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -25 $OUT/gpu_tests_$TAG.log
for c in 2 3; do
  ST=100; [ $c = 3 ] && ST=20
  SIDWT_TCS=1 timeout 300 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e --no-variants > $OUT/bench_${TAG}_c$c.json 2> $OUT/bench_${TAG}_c$c.err
  echo "C$c TCS"; python tools/bench_brief.py $OUT/bench_${TAG}_c$c.json; tail -3 $OUT/bench_${TAG}_c$c.err
done
