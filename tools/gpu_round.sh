# Full round measurement: build, smoke, GPU tests, bench (all configs), reference arm,
# launch list + one ncu full capture of the top kernel.  usage: bash tools/gpu_round.sh <tag>
TAG=${1:-r}; PART=${2:-main}     # main: tests, benches, reference, C2 ncu; c4 / c3: tensor-core kernel captures
OUT=gpurun_out
if [ "$PART" = main ]; then
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi_$TAG.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/gpu_tests_$TAG.log
timeout 600 python bench.py > $OUT/bench_${TAG}_c2.json 2> $OUT/bench_${TAG}_c2.err; echo "bench c2 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/ref_${TAG}_c2.json 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --config 3 --steps 20 > $OUT/bench_${TAG}_c3.json 2> $OUT/bench_${TAG}_c3.err; echo "bench c3 rc=$?"
timeout 600 python bench.py --config 5 --steps 20 > $OUT/bench_${TAG}_c5.json 2> $OUT/bench_${TAG}_c5.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --config 4 --steps 3 --no-e2e > $OUT/bench_${TAG}_c4.json 2> $OUT/bench_${TAG}_c4.err; echo "bench c4 rc=$?"
for c in c2 c3 c5 c4; do python tools/bench_brief.py $OUT/bench_${TAG}_$c.json; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variants"
timeout 300 $CMD > $OUT/plain_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_analyze|k_correlate" -s 4 -c 2 -o $OUT/prof_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"
fi
if [ "$PART" = c4 ]; then
# tensor-core bank kernel: launch list share and one full capture on a reduced C4 batch
CMD4="python bench.py --config 4 --rows 256 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-variants"
timeout 300 $CMD4 > $OUT/plain4_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches4_$TAG.csv $CMD4 > $OUT/ncu_launch4_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_correlate_tc|k_analyze" -s 2 -c 2 -o $OUT/prof4_$TAG $CMD4 > $OUT/ncu_full4_$TAG.log 2>&1
echo "ncu4 rc=$?"
fi
if [ "$PART" = c3 ]; then
CMD3="python bench.py --config 3 --rows 296 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-variants"
# single-template tensor-core kernel (C3): launch list and one full capture on a reduced batch
timeout 300 $CMD3 > $OUT/plain3_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $OUT/launches3_$TAG.csv $CMD3 > $OUT/ncu_launch3_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_correlate_tcs|k_analyze" -s 2 -c 2 -o $OUT/prof3_$TAG $CMD3 > $OUT/ncu_full3_$TAG.log 2>&1
echo "ncu3 rc=$?"
fi
