# sidwt_run chunk-count sweep: tests for the run path, then bench C2/C3/C5 per chunk count.
# usage: bash tools/gpu_run_sweep.sh <tag> "<chunk counts>" "<configs>"
TAG=${1:-rs}; CH=${2:-"1 2 4 8"}; CFGS=${3:-"2 3 5"}
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; tail $OUT/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "run or abi" > $OUT/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/gpu_tests_$TAG.log
for c in $CFGS; do
  ST=100; [ $c = 3 ] && ST=20; [ $c = 5 ] && ST=20; [ $c = 4 ] && ST=5
  for k in $CH; do
    SIDWT_RUN_CHUNKS=$k timeout 600 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e > $OUT/bench_${TAG}_c${c}_k$k.json 2> $OUT/bench_${TAG}_c${c}_k$k.err
    echo "C$c chunks=$k"; python tools/bench_brief.py $OUT/bench_${TAG}_c${c}_k$k.json
  done
done
