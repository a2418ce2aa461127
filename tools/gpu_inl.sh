OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_inl.log 2>&1 || { echo build failed; exit 1; }
SIDWT_K2_INLINE=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_run.py -m gpu -q -x > $OUT/gpu_tests_inl.log 2>&1; echo "tests(inline) rc=$?"; tail -2 $OUT/gpu_tests_inl.log | cut -c1-300
for V in SIDWT_K2_INLINE=0 SIDWT_K2_INLINE=1; do for c in 2 5; do
  ST=100; [ $c = 5 ] && ST=20
  env $V timeout 300 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e > $OUT/b_c$c.json 2>/dev/null
  echo "[$V] C$c"; python tools/bench_brief.py $OUT/b_c$c.json | cut -c1-200
done; done
