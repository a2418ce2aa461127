# sweep env knobs on the C2 bench. usage: bash tools/gpu_sweep.sh <tag> "<VAR=a VAR2=b>" ...
TAG=$1; shift
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1 || { echo build failed; exit 1; }
for V in "$@"; do
  env $V timeout 300 python bench.py --steps 100 --no-cpu-baseline --no-e2e $BENCH_ARGS > $OUT/sweep_$TAG.json 2>&1
  python -c "import json,sys; d=json.loads(open('$OUT/sweep_$TAG.json').read().strip().splitlines()[-1]); s=d['stages']; print('$V', '| ms/step %.3f'%d['ms_per_step'], 'analyze %.3f ms %.0f GB/s'%(s['analyze']['ms'], s['analyze']['achieved']), 'corr %.3f ms %.1f TF'%(s['correlate_peaks']['ms'], s['correlate_peaks']['alu']['achieved']))" || tail -3 $OUT/sweep_$TAG.json
done
