OUT=gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "5 or int or random or fused or run" > $OUT/gpu_tests_c5q.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/gpu_tests_c5q.log
timeout 300 python bench.py --config 5 --steps 20 --no-cpu-baseline --no-e2e --no-variants > $OUT/b.json 2>/dev/null
python -c "import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); s=d['stages']; print('C5 step %.3f corr %.3f'%(d['ms_per_step'], s['correlate_peaks']['ms']))"
