# ncu full capture of the 3xTF32 tcgen05 gemm at 16384^3 (one launch) -> gpurun_out/gemm_full.ncu-rep
python tools/gemm_probe.py > gpurun_out/gemm_probe.txt 2>&1; echo probe=$?
ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32 -c 1 -o gpurun_out/gemm_full \
    python tools/gemm_probe.py > gpurun_out/gemm_ncu.log 2>&1; echo ncu=$?
ncu -i gpurun_out/gemm_full.ncu-rep --page raw --csv > gpurun_out/gemm_raw.csv 2>&1
