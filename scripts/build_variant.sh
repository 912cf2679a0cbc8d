#!/bin/bash
# Build a variant of libb3d_b200.so with extra nvcc defines for same-box A/B:
#   scripts/build_variant.sh NAME -DFOO=1 ...   -> _ab/lib_NAME.so
NAME=$1; shift
cd "$(dirname "$0")/.."
make -s -j8 -C paper_2312_08715_b200/csrc >/dev/null 2>&1 || exit 1
T=$(mktemp -d)
C=paper_2312_08715_b200/csrc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xptxas -v -Xcompiler -fPIC,-fvisibility=hidden,-O2 -Iinclude -I$C"
for f in render_score rs_score_w0 rs_score_w1 rs_score_w2 rs_score_w3 rs_score_wx rs_cam rs_cam_w1 rs_cam_w2 rs_cam_w4; do
  /usr/local/cuda/bin/nvcc $FL "$@" -c $C/$f.cu -o $T/$f.o 2> $T/$f.log &
done
wait
grep -h "spill" $T/rs_score_w1.log | head -1
O=build/obj
mkdir -p _ab
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o _ab/lib_$NAME.so \
  $T/*.o $O/stage.cu.o $O/image_score.cu.o $O/exact_score.cu.o $O/exchange.cu.o $O/mesh_build.cu.o $O/track.cu.o $O/b3d_capi.cpp.o $O/smc.cpp.o $O/capi_handles.cpp.o -Xlinker --no-undefined -lpthread -ldl -lrt || cat $T/*.log
rm -rf $T
