# build the working tree's library with extra nvcc flags into _lib/librangeseg_b200_$1.so
set -e
NAME=$1; shift
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC -shared -cudart static "$@" -I /root/repo/include -o /root/repo/paper_2003_00575_b200/_lib/librangeseg_b200_$NAME.so /root/repo/paper_2003_00575_b200/csrc/rangeseg_b200.cu
