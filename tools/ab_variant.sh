# Build an A/B variant of one translation unit: tools/ab_variant.sh <name> <unit.cu> [unit basename to replace] [extra nvcc flags]
# -> abtmp/libsidwt_<name>.so (the other objects come from build/)
NAME=$1; SRC=$2; UNIT=${3:-corr_i8}; EXTRA=$4
mkdir -p abtmp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Ipaper_cs_0607001_b200/csrc $EXTRA -c -o abtmp/${UNIT}_$NAME.o $SRC || exit 1
OBJS=$(ls build/*.o | grep -v "/$UNIT.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o abtmp/libsidwt_$NAME.so $OBJS abtmp/${UNIT}_$NAME.o
