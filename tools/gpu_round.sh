# Round measurement on one B200 (run under gpurun from the repo root).
#   bash tools/gpu_round.sh <tag> main   : build, smoke, GPU tests, bench lines C5 (default) / C2 / C3 / C4, reference arm
#   bash tools/gpu_round.sh <tag> ncu    : launch list of the default bench command + one ncu --set full capture
#                                          of the two kernels of the C5 step (reduced batch; traffic scales with rows)
#   bash tools/gpu_round.sh <tag> ncu3|ncu4|ncu2 : the same for C3 / C4 / C2
#   bash tools/gpu_round.sh <tag> san <tool>     : compute-sanitizer <tool> over tests/test_gpu_sanitize.py
TAG=${1:-r}; PART=${2:-main}
OUT=gpurun_out
mkdir -p $OUT
if [ "$PART" = main ]; then
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi_$TAG.txt
  python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 $OUT/smoke_$TAG.log
  timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -4 $OUT/gpu_tests_$TAG.log
  timeout 900 python bench.py > $OUT/bench_${TAG}_c5.json 2> $OUT/bench_${TAG}_c5.err; echo "bench c5 rc=$?"
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref_${TAG}_c5.json 2>&1; echo "ref rc=$?"
  timeout 600 python bench.py --config 2 > $OUT/bench_${TAG}_c2.json 2> $OUT/bench_${TAG}_c2.err; echo "bench c2 rc=$?"
  timeout 900 python bench.py --config 3 --steps 20 > $OUT/bench_${TAG}_c3.json 2> $OUT/bench_${TAG}_c3.err; echo "bench c3 rc=$?"
  timeout 1500 python bench.py --config 4 --steps 3 --no-e2e > $OUT/bench_${TAG}_c4.json 2> $OUT/bench_${TAG}_c4.err; echo "bench c4 rc=$?"
  for c in c5 c2 c3 c4; do python tools/bench_brief.py $OUT/bench_${TAG}_$c.json; done
fi
ncu_pair() {   # $1 suffix, $2 config, $3 rows for the full capture, $4 kernel regex
  CMD="python bench.py --config $2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variants"
  CMDR="$CMD --rows $3"
  timeout 600 $CMD > $OUT/plain$1_$TAG.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches$1_$TAG.csv $CMD > $OUT/ncu_launch$1_$TAG.log 2>&1 && \
  timeout 300 $CMDR > $OUT/plainr$1_$TAG.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$4" -s 1 -c 1 -o $OUT/prof$1_$TAG $CMDR > $OUT/ncu_full$1_$TAG.log 2>&1
  echo "ncu$1 rc=$?"
}
[ "$PART" = ncu ] && ncu_pair 5 5 4096 "k_correlate"
[ "$PART" = ncu2 ] && ncu_pair 2 2 4096 "k_correlate"
[ "$PART" = ncu3 ] && ncu_pair 3 3 296 "k_correlate"
[ "$PART" = ncu4 ] && ncu_pair 4 4 256 "k_correlate_tc"
[ "$PART" = ncuA ] && ncu_pair A${3:-5} ${3:-5} ${4:-4096} "k_analyze"
if [ "$PART" = san ]; then
  TOOL=${3:-memcheck}
  timeout 1800 compute-sanitizer --tool $TOOL --error-exitcode 99 python -m pytest -q -x tests/test_gpu_sanitize.py \
     > $OUT/sanitize_${TOOL}_$TAG.log 2>&1
  echo "sanitize $TOOL rc=$?"; tail -5 $OUT/sanitize_${TOOL}_$TAG.log
fi
