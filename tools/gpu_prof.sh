# usage: bash tools/gpu_prof.sh <tag> [bench-args...]
TAG=${1:-r1}; shift
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; tail $OUT/build_$TAG.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -5 $OUT/gpu_tests_$TAG.log
timeout 600 python bench.py "$@" > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -c 3000 $OUT/bench_$TAG.json
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $@"
timeout 300 $CMD > $OUT/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_analyze|k_correlate" -s 4 -c 2 -o $OUT/prof_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"; tail -3 $OUT/ncu_full_$TAG.log
