# ncu --set full of the device-fit kernels at the C3 shape (2048 x 5504, d = 1024, T = 9):
# the batched fp64 gather (largest launch), the fused trial tile kernels, and the DMMA GEMM.
mkdir -p gpurun_out
rm -f gpurun_out/prof_fit_*.ncu-rep
timeout 900 ncu --set full --clock-control none -k "regex:k_gather_f64v" -s 200 -c 1 -o gpurun_out/prof_fit_gather python tools/fitcap.py 9 2048 5504 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k "regex:k_poly_tile|k_dot_tile" -s 10 -c 2 -o gpurun_out/prof_fit_tiles python tools/fitcap.py 9 2048 5504 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k "regex:k_dgemm" -c 1 -o gpurun_out/prof_fit_dgemm python tools/prof_reproject.py > /dev/null 2>&1
ls gpurun_out/prof_fit_*
