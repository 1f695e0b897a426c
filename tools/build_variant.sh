#!/bin/bash
# Build a predictor variant library for A/B timing (tools/pred_ab.py):
#   tools/build_variant.sh NAME "-DMACRO=VAL ..." [SOURCE (default adg_predictor)]
# Output: paper_1808_03788_b200/variants/libNAME.so (git-ignored, travels with gpurun).
set -e
cd "$(dirname "$0")/.."
make -C paper_1808_03788_b200/csrc -j8 >/dev/null
mkdir -p build/variants paper_1808_03788_b200/variants
NV=/usr/local/cuda/bin/nvcc
SRC=${3:-adg_predictor}
FL="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -rdc=true -Xcompiler -fPIC,-O2 -Xptxas -v --expt-relaxed-constexpr"
(cd paper_1808_03788_b200/csrc && $NV $FL $2 -c $SRC.cu -o ../../build/variants/pred_$1.o 2> ../../build/variants/pred_$1.log)
$NV -gencode arch=compute_100a,code=sm_100a -rdc=true -shared -Xcompiler -fPIC \
  $(ls build/obj/*.o | grep -v "$SRC.o") build/variants/pred_$1.o \
  -o paper_1808_03788_b200/variants/lib$1.so -ldl
python tools/ptxas_regs.py build/variants/pred_$1.log "predict_kernel<3, 5, 0>" 2>/dev/null || true
