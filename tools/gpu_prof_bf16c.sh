# ncu --set full of the bf16 gather compress (C4-bf16 and C3, layer 8) and the fp32 one for comparison.
mkdir -p gpurun_out/pbf
for c in c4-bf16 c3; do
timeout 600 ncu --set full --clock-control none -k regex:k_compress_spmm -s 8 -c 1 -o gpurun_out/pbf/spmm_$c python bench.py --config $c --fit-every 0 --steps 1 --warmup 1 --graph 0 --no-e2e --no-cpu-baseline > /dev/null 2>gpurun_out/pbf/$c.err; tail -1 gpurun_out/pbf/$c.err
python tools/ncu_stalls.py gpurun_out/pbf/spmm_$c.ncu-rep 2>&1 | head -30
done
