# k_build_y_vec columns-per-warp variants (rebuilds the library on the box)
mkdir -p gpurun_out
F=paper_2406_10181_b200/csrc/apply.cu
run() {
  make -C paper_2406_10181_b200/csrc -j16 > gpurun_out/mk.log 2>&1 || { echo "build failed $1"; tail -3 gpurun_out/mk.log; return; }
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1', round(d['ms_per_step'],3), 'build', round(b['build_y_ms_per_step'],3))" || tail -2 gpurun_out/b.err
}
run base8
sed -i "s/^constexpr int kYVJ = [0-9]*;/constexpr int kYVJ = 4;/" $F; run yvj4
