# build_y_vec columns-per-warp sweep (rebuilds the library on the box for each value)
mkdir -p gpurun_out
for v in 4 16 8; do
  sed -i "s/^constexpr int kYVJ = [0-9]*;/constexpr int kYVJ = $v;/" paper_2406_10181_b200/csrc/apply.cu
  make -C paper_2406_10181_b200/csrc -j16 > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('kYVJ=$v', round(d['ms_per_step'],3), round(b['build_y_ms_per_step'],3))" || tail -2 gpurun_out/b.err
done
