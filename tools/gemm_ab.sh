# A/B timing of gemm builds (default + variants/<name> given as arguments) at 8192^3 and 16384^3
for v in default "$@"; do
  if [ $v = default ]; then L=""; else L=variants/$v/libpencil_b200.so; fi
  echo "$v 8192: $(PENCIL_B200_LIB=$L timeout 120 python tools/gemm_probe.py 8192 2>&1 | tail -1)"
  echo "$v 16384: $(PENCIL_B200_LIB=$L timeout 120 python tools/gemm_probe.py 16384 2>&1 | tail -1)"
done
