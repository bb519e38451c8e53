# Build a library variant from the working tree with a sed expression applied to one
# source file: tools/ab_build.sh <out.so> <file.cu> '<sed expr>'
set -e
T=$(mktemp -d)
mkdir -p $T/p/csrc $T/include
cp paper_2403_19272_b200/csrc/* $T/p/csrc/
cp include/*.h $T/include/
sed -i "$3" $T/p/csrc/$2
(cd $T/p/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC,-Wno-deprecated-declarations -shared abi.cu -o $T/out.so)
cp $T/out.so $1
rm -rf $T
