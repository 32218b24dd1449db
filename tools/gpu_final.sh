# Final capture of the round: every GPU test, smoke, the default bench line and
# the reference arm (gpu_validate.sh), then the C4 ncu launch list + --set full
# of the step kernels (gpu_profile_kernels.sh) on the same sources.
bash tools/gpu_validate.sh
bash tools/gpu_profile_kernels.sh
