# On the GPU box after tools/gpu_round.sh <tag> ncu*: turn the captures into the small text summaries that
# travel back (the .ncu-rep files are removed: gpurun_out/ is limited to 64 MiB).
#   bash tools/gpu_profiles.sh <tag>
TAG=$1; OUT=gpurun_out
for f in $OUT/prof*_$TAG.ncu-rep; do
  [ -f "$f" ] || continue
  b=$(basename $f .ncu-rep)
  python tools/ncu_summary.py $f > $OUT/${b}_summary.txt 2>&1
  python tools/sass_hot.py $f 1.0 > $OUT/${b}_hot.txt 2>&1
done
[ -f $OUT/prof5_$TAG.ncu-rep ] && python tools/ncu_traffic.py $OUT/prof5_$TAG.ncu-rep C5_4096rows
[ -f $OUT/profA5_$TAG.ncu-rep ] && python tools/ncu_traffic.py $OUT/profA5_$TAG.ncu-rep C5_4096rows
[ -f $OUT/prof3_$TAG.ncu-rep ] && python tools/ncu_traffic.py $OUT/prof3_$TAG.ncu-rep C3_296rows
cp profiles/ncu_traffic.json $OUT/ncu_traffic_$TAG.json
for c in 5 3 4 2; do
  [ -f $OUT/launches${c}_$TAG.csv ] && python tools/launch_summary.py $OUT/launches${c}_$TAG.csv "C$c bench command, $TAG" > $OUT/launches${c}_${TAG}_summary.txt
done
rm -f $OUT/*.ncu-rep
