# TC path check: build, small TC tests (short timeout), then full-size + C4 bench variants.
# usage: bash tools/gpu_tc.sh <tag> "<env settings for variants>"...
TAG=${1:-tc}; shift
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; tail $OUT/build_$TAG.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_tc.py -q -x -k "not full_size" > $OUT/tc_tests_$TAG.log 2>&1; rc=$?
echo "tc small tests rc=$rc"; tail -30 $OUT/tc_tests_$TAG.log | cut -c1-400
[ $rc = 0 ] || exit 1
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x -k "full_size" -s > $OUT/tc_full_$TAG.log 2>&1; echo "tc full rc=$?"; tail -5 $OUT/tc_full_$TAG.log | cut -c1-400
for V in "$@"; do
  env $V timeout 600 python bench.py --config 4 --steps 5 --no-cpu-baseline --no-e2e > $OUT/bench_${TAG}_c4.json 2> $OUT/bench_${TAG}_c4.err
  echo "[$V]"; python tools/bench_brief.py $OUT/bench_${TAG}_c4.json; tail -3 $OUT/bench_${TAG}_c4.err
done
