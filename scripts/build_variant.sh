# build the library of git revision $1 into paper_2003_00575_b200/_lib/librangeseg_b200_$2.so
set -e
REV=$1; NAME=$2
TMP=$(mktemp -d)
git -C /root/repo archive $REV paper_2003_00575_b200/csrc include | tar -x -C $TMP
mkdir -p $TMP/paper_2003_00575_b200/_lib
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC -shared -cudart static -I $TMP/include -o /root/repo/paper_2003_00575_b200/_lib/librangeseg_b200_$NAME.so $TMP/paper_2003_00575_b200/csrc/rangeseg_b200.cu
rm -rf $TMP
