# A/B of the stage-2 + Adam fusion (C4 fp32): bench lines and ncu launch times
B="python bench.py --no-e2e --no-cpu-baseline"
timeout 600 python -m pytest tests/test_gpu_fused_adam.py -x -q > gpurun_out/t2.log 2>&1
for R in 1 2 4; do LSP_S2A_ROWS=$R timeout 300 $B > gpurun_out/b_r$R.json 2> gpurun_out/b_r$R.err; done
LSP_FUSE_ADAM=0 timeout 300 $B > gpurun_out/b_unf.json 2> gpurun_out/b_unf.err
timeout 300 $B > gpurun_out/b_r1b.json 2> gpurun_out/b_r1b.err
for V in fused unf; do
  E=""; [ $V = unf ] && E="LSP_FUSE_ADAM=0"
  env $E timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_stage2|k_adam' -c 40 --csv \
    --log-file gpurun_out/ncu_$V.csv python bench.py --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_$V.log 2>&1
done
tail -2 gpurun_out/t2.log
