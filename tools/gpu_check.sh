# build, GPU tests (optional -k filter), brief benches of the given configs.
# usage: bash tools/gpu_check.sh <tag> "<pytest -k expr or empty>" "<configs, e.g. 2 3 5>" [extra bench args]
TAG=${1:-q}; K=${2:-}; CFGS=${3:-2}; shift 3; EXTRA="$@"
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; tail $OUT/build_$TAG.log; exit 1; }
if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > $OUT/gpu_tests_$TAG.log 2>&1; else timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/gpu_tests_$TAG.log 2>&1; fi
echo "tests rc=$?"; tail -4 $OUT/gpu_tests_$TAG.log
for c in $CFGS; do
  ST=100; [ $c = 3 ] && ST=20; [ $c = 5 ] && ST=20; [ $c = 4 ] && ST=5
  timeout 600 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e $EXTRA > $OUT/bench_${TAG}_c$c.json 2> $OUT/bench_${TAG}_c$c.err
  python tools/bench_brief.py $OUT/bench_${TAG}_c$c.json
done
