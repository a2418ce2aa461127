# ncu full capture of the TC correlation kernel on a reduced C4 batch. usage: bash tools/gpu_ncu_tc.sh <tag> [env]
TAG=${1:-p}; shift
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
CMD="python bench.py --config 4 --rows 256 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
env "$@" timeout 300 $CMD > $OUT/plain_$TAG.log 2>&1 && \
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_correlate_tc" -s 2 -c 1 -o $OUT/prof_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"; tail -3 $OUT/ncu_full_$TAG.log
