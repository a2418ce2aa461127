OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 5 2 3; do for L in 2048 3072 4096 6144; do
  ST=100; [ $c = 3 ] && ST=20; [ $c = 5 ] && ST=20
  SIDWT_K1_LBUF=$L timeout 300 python bench.py --config $c --steps $ST --no-cpu-baseline --no-e2e --no-variants > $OUT/b.json 2>/dev/null
  python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); a=d['stages']['analyze']; print('C$c lbuf=$L analyze %.3f ms %.0f%%'%(a['ms'], 100*a['frac']))"
done; done
