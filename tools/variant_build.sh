#!/bin/bash
# A/B builds of the product library: the shipped .so carries no run-time selection knobs; each
# measured alternative is a compile-time variant built here into variants/<name>/ and loaded with
# PENCIL_B200_LIB=variants/<name>/libpencil_b200.so (tools/ab_spmv.sh, bench.py).
#   bash tools/variant_build.sh <name> -DPENCIL_VARIANT_...
# Known variants:
#   -DPENCIL_VARIANT_NO_SWAR     packed-byte stencil without the 16-bit SWAR kernel
#   -DPENCIL_VARIANT_SWAR_NP8    SWAR kernel at 8 px per lane only
#   -DPENCIL_VARIANT_NO_SEP      no separable (rank-1) stencil kernels
#   -DPENCIL_VARIANT_NO_DIA      no diamond-support stencil kernels
#   -DPENCIL_VARIANT_NO_PF       no power-of-two fused f32 taps
#   -DPENCIL_VARIANT_L2_DIRTY    L2 flush without the discard (dirty lines left)
#   -DPENCIL_VARIANT_NO_SEG      spmv_vec on the batch-and-fold executor (csr_flow_kernel), not csr_seg_kernel
#   -DGEMM_LO_TRUNC              gemm lo halves truncated by the tensor core instead of rounded (timing only)
#   -DGEMM_LO_CVT                gemm lo halves rounded by cvt.rna.tf32 (round 2's first form; same bits)
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
make -s -j8 -C "$root/paper_1302_5586_b200" VARIANT="$*" BUILD="$root/variants/$name/build" \
     LIBDIR="$root/variants/$name" "$root/variants/$name/libpencil_b200.so"
echo "variants/$name/libpencil_b200.so ($*)"
