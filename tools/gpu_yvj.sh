# build_y_vec variants (rebuilds the library on the box for each)
mkdir -p gpurun_out
F=paper_2406_10181_b200/csrc/apply.cu
run() {
  make -C paper_2406_10181_b200/csrc -j16 > gpurun_out/mk.log 2>&1 || { echo "build failed $1"; tail -3 gpurun_out/mk.log; return; }
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1', round(d['ms_per_step'],3), round(b['build_y_ms_per_step'],3))" || tail -2 gpurun_out/b.err
}
sed -i "s/^constexpr int kYVJ = [0-9]*;/constexpr int kYVJ = 4;/" $F; run yvj4
sed -i "s/^constexpr int kYVJ = [0-9]*;/constexpr int kYVJ = 8;/" $F
sed -i "s/__launch_bounds__(256) k_build_y_vec/__launch_bounds__(256, 2) k_build_y_vec/" $F; run lb2
sed -i "s/__launch_bounds__(256, 2) k_build_y_vec/__launch_bounds__(256, 6) k_build_y_vec/" $F; run lb6
sed -i "s/__launch_bounds__(256, 6) k_build_y_vec/__launch_bounds__(256) k_build_y_vec/" $F; run base
