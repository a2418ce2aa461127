# On the GPU box: time the default bench with each abtmp/libsidwt_<name>.so swapped in.
#   bash tools/ab_run.sh "<bench args>" name1 name2 ...
ARGS=$1; shift
cp paper_cs_0607001_b200/libsidwt.so abtmp/libsidwt__keep.so
for n in "$@" "$@"; do
  cp abtmp/libsidwt_$n.so paper_cs_0607001_b200/libsidwt.so
  timeout 600 python bench.py $ARGS --no-cpu-baseline --no-e2e --no-variants > gpurun_out/ab_$n.json 2> gpurun_out/ab_$n.err
  echo -n "$n: "; python tools/bench_brief.py gpurun_out/ab_$n.json | head -1
done
cp abtmp/libsidwt__keep.so paper_cs_0607001_b200/libsidwt.so
