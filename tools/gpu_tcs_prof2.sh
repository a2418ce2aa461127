OUT=gpurun_out
SIDWT_TC_PROFILE=1 python -c "from paper_cs_0607001_b200 import _native; _native.build(force=True)" > $OUT/build_prof.log 2>&1 || { echo build failed; tail $OUT/build_prof.log; exit 1; }
for pr in 1 3; do for c in 3 2; do
  SIDWT_TCS=1 SIDWT_TC_PROF=$pr timeout 300 python bench.py --config $c --rows 296 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > $OUT/tcsprof_c$c.log 2>&1
  echo "C$c prof=$pr"; grep "tcs cta0" $OUT/tcsprof_c$c.log | tail -4
done; done
python -c "from paper_cs_0607001_b200 import _native; _native.build(force=True)" > /dev/null 2>&1
for c in 2 3; do
  ST=100; [ $c = 3 ] && ST=20
  SIDWT_TCS=1 timeout 300 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e --no-variants > $OUT/b_c$c.json 2>/dev/null
  echo "C$c TCS"; python tools/bench_brief.py $OUT/b_c$c.json
done
