# Sweep the segmented executor's compile-time shape (tile non-zeros x non-zeros per lane x CTAs per
# SM) for both SpMV modes: each point is a variant build (tools/variant_build.sh), timed with
# tools/ab_spmv_modes.sh on one box.  Round-1 form of this sweep used run-time knobs; the shipped
# library has none.
#   bash tools/spmv_sweep.sh          (builds variants/*, then: gpurun -- 'bash tools/ab_spmv_modes.sh base t2048 ...')
set -e
for T in 2048 4096 8192; do bash tools/variant_build.sh t$T -DSEG_TILE_NNZ=$T > /dev/null; echo "variants/t$T"; done
for C in 4 5 6; do bash tools/variant_build.sh c$C -DSEG_CTAS_PER_SM=$C > /dev/null; echo "variants/c$C"; done
for E in 4 8; do bash tools/variant_build.sh oe$E -DSEG_E_ORD=$E > /dev/null; echo "variants/oe$E"; done
