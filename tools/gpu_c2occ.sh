OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for V in "SIDWT_K2_MINB=3" "SIDWT_K2_MINB=3 SIDWT_K2_NBUF=1" "SIDWT_K2_MINB=4 SIDWT_K2_NBUF=1"; do
  env $V timeout 300 python bench.py --config 2 --steps 200 --no-cpu-baseline --no-e2e --no-variants > $OUT/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); s=d['stages']; print('[$V] step %.4f corr %.4f'%(d['ms_per_step'], s['correlate_peaks']['ms']))"
done
