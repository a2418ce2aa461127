# ncu full capture of one kernel from a short bench run. usage: bash tools/gpu_ncu.sh <tag> <kernel regex> [bench args...]
TAG=$1; KRE=$2; shift 2
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $@"
timeout 300 $CMD > $OUT/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 2 -c 1 -o $OUT/prof_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"; tail -2 $OUT/ncu_full_$TAG.log
