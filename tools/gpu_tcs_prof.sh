# timed role waits of k_correlate_tcs (CTA 0), reduced C2/C3 batches
OUT=gpurun_out
SIDWT_TC_PROFILE=1 python -c "from paper_cs_0607001_b200 import _native; _native.build(force=True)" > $OUT/build_prof.log 2>&1 || { echo build failed; tail $OUT/build_prof.log; exit 1; }
for c in 3 2; do
  SIDWT_TCS=1 SIDWT_TC_PROF=1 timeout 300 python bench.py --config $c --rows 296 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > $OUT/tcsprof_c$c.log 2>&1
  echo "C$c"; grep "tcs cta0" $OUT/tcsprof_c$c.log | tail -4
done
