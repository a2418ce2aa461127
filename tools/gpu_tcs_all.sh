# TCS: tests, role-wait profile (C3/C2 reduced), benches C2/C3 (SIDWT_TCS=1)
TAG=${1:-tcs}
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; tail $OUT/build_$TAG.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_tcs.py -m gpu -q -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -4 $OUT/gpu_tests_$TAG.log | cut -c1-300
for c in 2 3; do
  ST=100; [ $c = 3 ] && ST=20
  SIDWT_TCS=1 timeout 300 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e --no-variants > $OUT/bench_${TAG}_c$c.json 2> $OUT/bench_${TAG}_c$c.err
  echo "C$c TCS"; python tools/bench_brief.py $OUT/bench_${TAG}_c$c.json
done
SIDWT_TC_PROFILE=1 python -c "from paper_cs_0607001_b200 import _native; _native.build(force=True)" > $OUT/build_prof.log 2>&1
for c in 3 2; do
  SIDWT_TCS=1 SIDWT_TC_PROF=1 timeout 300 python bench.py --config $c --rows 296 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > $OUT/tcsprof_c$c.log 2>&1
  echo "C$c prof"; grep "tcs cta0" $OUT/tcsprof_c$c.log | tail -4
done
python -c "from paper_cs_0607001_b200 import _native; _native.build(force=True)" > /dev/null 2>&1
