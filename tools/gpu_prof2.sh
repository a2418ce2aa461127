# tests + bench + ncu full capture of k_correlate only. usage: bash tools/gpu_prof2.sh <tag> [bench args]
TAG=${1:-p}; shift
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/gpu_tests_$TAG.log
timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e "$@" > $OUT/bench_$TAG.json 2>&1
python -c "import json,sys; d=json.loads(open('$OUT/bench_$TAG.json').read().strip().splitlines()[-1]); s=d['stages']; print('ms/step %.3f'%d['ms_per_step'], 'analyze %.3f ms %.0f GB/s'%(s['analyze']['ms'], s['analyze']['achieved']), 'corr %.3f ms %.1f TF'%(s['correlate_peaks']['ms'], s['correlate_peaks']['alu']['achieved']), d['clocks'])"
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $@"
timeout 300 $CMD > $OUT/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_analyze|k_correlate" -s 4 -c 2 -o $OUT/prof_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu rc=$?"
