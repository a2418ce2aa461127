# ncu full capture of k_correlate_tcs on a reduced batch. usage: bash tools/gpu_ncu_tcs.sh <tag> <config> <rows>
TAG=$1; C=${2:-3}; R=${3:-296}
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
CMD="python bench.py --config $C --rows $R --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-variants"
SIDWT_TCS=1 timeout 300 $CMD > $OUT/plain_$TAG.log 2>&1 && python tools/bench_brief.py $OUT/plain_$TAG.log
SIDWT_TCS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_correlate_tcs" -s 2 -c 1 -o $OUT/prof_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"; tail -2 $OUT/ncu_full_$TAG.log
