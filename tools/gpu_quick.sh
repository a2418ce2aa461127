# quick: build, gpu tests (optionally filtered), bench variants. usage: bash tools/gpu_quick.sh <tag> [pytest -k expr]
TAG=${1:-q}; K=${2:-}
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; tail $OUT/build_$TAG.log; exit 1; }
if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -q -x -k "$K" > $OUT/gpu_tests_$TAG.log 2>&1; else timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/gpu_tests_$TAG.log 2>&1; fi
echo "tests rc=$?"; tail -4 $OUT/gpu_tests_$TAG.log
for TT in 2048 1024; do
 SIDWT_K2_TT=$TT timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e > $OUT/bench_${TAG}_tt$TT.json 2>&1
 python -c "import json,sys; d=json.loads(open('$OUT/bench_${TAG}_tt$TT.json').read().strip().splitlines()[-1]); s=d['stages']; print('TT=$TT', 'ms/step %.3f'%d['ms_per_step'], 'analyze %.3f ms %.0f GB/s'%(s['analyze']['ms'], s['analyze']['achieved']), 'corr %.3f ms %.1f TF'%(s['correlate_peaks']['ms'], s['correlate_peaks']['alu']['achieved']), d['clocks'])"
done
