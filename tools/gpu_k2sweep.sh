OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 2 5; do for T in 1024 2048 4096; do for MB in 2 3; do
  ST=100; [ $c = 5 ] && ST=20
  SIDWT_K2_TT=$T SIDWT_K2_MINB=$MB timeout 300 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e --no-variants > $OUT/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); a=d['stages']['correlate_peaks']; print('C$c TT=$T minb=$MB corr %.3f ms'%(a['ms']))"
done; done; done
