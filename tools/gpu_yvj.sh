# build_y_vec store-policy variants (rebuilds the library on the box for each)
mkdir -p gpurun_out
F=paper_2406_10181_b200/csrc/apply.cu
run() {
  make -C paper_2406_10181_b200/csrc -j16 > gpurun_out/mk.log 2>&1 || { echo "build failed $1"; tail -3 gpurun_out/mk.log; return; }
  timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
  python -c "import json;d=json.load(open('gpurun_out/b.json'));b=d['breakdown'];print('$1', round(d['ms_per_step'],3), 'build', round(b['build_y_ms_per_step'],3), 'apply', round(b['apply_ms_per_step'],3))" || tail -2 gpurun_out/b.err
}
run base
cp $F /tmp/apply.cu.bak
sed -i '363s/, pol_last);/, policy_evict_first());/' $F; run evict_first
cp /tmp/apply.cu.bak $F
python - <<'PY'
p='paper_2406_10181_b200/csrc/apply.cu'; s=open(p).read()
a="""      st_hint_f4(reinterpret_cast<float*>(o + t / 4),
                 make_float4(y[t][c], y[t + 1][c], y[t + 2][c], y[t + 3][c]), pol_last);"""
b="""      o[t / 4] = make_float4(y[t][c], y[t + 1][c], y[t + 2][c], y[t + 3][c]);"""
assert a in s; s=s.replace(a,b,1); open(p,'w').write(s)
PY
run plain
cp /tmp/apply.cu.bak $F
