OUT=gpurun_out
SIDWT_TC_PROFILE=1 python -c "from paper_cs_0607001_b200 import _native; _native.build(force=True)" > $OUT/build_prof.log 2>&1 || { echo build failed; tail $OUT/build_prof.log; exit 1; }
for pr in 1 5; do
  SIDWT_TC_PROF=$pr timeout 300 python bench.py --config 3 --rows 296 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > $OUT/tcsprof.log 2>&1
  echo "C3 prof=$pr"; grep "tcs cta0" $OUT/tcsprof.log | tail -4
done
python -c "from paper_cs_0607001_b200 import _native; _native.build(force=True)" > /dev/null 2>&1
