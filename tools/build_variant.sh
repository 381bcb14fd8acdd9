#!/bin/bash
# Build an A/B variant of the device library with extra nvcc defines:
#   tools/build_variant.sh <out.so> -DQSB_GEMM_STAGES_256=4 -DQSB_GEMM_EPIBUFS_256=2
# Run with QSYNC_B200_LIB=<out.so> (paper_2407_02327_b200/_lib.py).
set -e
out=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
tmp=$(mktemp -d)
srcs=$(ls $root/paper_2407_02327_b200/csrc/*.cu $root/paper_2407_02327_b200/csrc/*.cpp)
for s in $srcs; do
  b=$(basename $s); o=$tmp/${b%.*}.o
  if [[ $s == *.cu ]]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 \
      --expt-relaxed-constexpr -I$root/include -I$root/paper_2407_02327_b200/csrc "$@" -c $s -o $o &
  else
    g++ -O2 -std=c++17 -fPIC -mpclmul -msse4.1 -I$root/include -I$root/paper_2407_02327_b200/csrc -c $s -o $o &
  fi
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out $tmp/*.o
rm -rf $tmp
echo built $out
