# build an experimental variant of libexg.so with extra nvcc defines:
#   bash tools/build_variant.sh NAME "-DFOO -DBAR=1"   -> exp/NAME/libexg.so
# select it at run time with EXG_LIB=exp/NAME/libexg.so
set -e
NAME=$1; DEFS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_1511_04515_b200/csrc
NV="-gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -fmad=false --extended-lambda -Xcompiler -fPIC,-ffp-contract=off -I$ROOT/include -I$C $DEFS"
mkdir -p $ROOT/exp/$NAME
make -s -j8 -C $C OUT=$ROOT/exp/$NAME/libexg.so BUILD=$ROOT/build/exg_$NAME NVFLAGS="$NV"
