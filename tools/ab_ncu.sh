# On the GPU box: one ncu --set full capture (source-level) of a kernel with abtmp/libsidwt_<name>.so swapped in.
#   bash tools/ab_ncu.sh <kernel regex> "<bench args>" name1 name2 ...
KRE=$1; ARGS=$2; shift; shift
cp paper_cs_0607001_b200/libsidwt.so abtmp/libsidwt__keep.so
for n in "$@"; do
  cp abtmp/libsidwt_$n.so paper_cs_0607001_b200/libsidwt.so
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 1 -c 1 -f -o gpurun_out/prof_$n \
    python bench.py $ARGS --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/ncu_$n.log 2>&1
  echo "$n rc=$?"
done
cp abtmp/libsidwt__keep.so paper_cs_0607001_b200/libsidwt.so
