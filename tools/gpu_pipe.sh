# Pipelined schedule (stage 2 + Adam beside the next layer's Y build): bitwise check + C4/bf16/C3.
mkdir -p gpurun_out
cat > /tmp/pipe_check.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2406_10181_b200 as lsp
from paper_2406_10181_b200.schedule import LayerSchedule
sys.path.insert(0, "tests")
import test_gpu_schedule as T
for mode in (1, 2):
    la, wa = T._build(); lb, wb = T._build()
    sa = LayerSchedule(la, 1e-3); sb = LayerSchedule(lb, 1e-3, pipeline=mode)
    for _ in range(3):
        sa.step(); sb.step()
    torch.cuda.synchronize()
    print("pipeline", mode, "bitwise", all(torch.equal(x, y) for x, y in zip(wa, wb)))
PY
python /tmp/pipe_check.py
for c in c4 c4-bf16 c3; do for p in 0 1 2; do
timeout 600 python bench.py --config $c --pipeline $p --schedule python --no-e2e --no-cpu-baseline --fit-every 0 > gpurun_out/pp.json 2> gpurun_out/pp.err
python -c "
import json;d=json.load(open('gpurun_out/pp.json'));print('$c pipeline=$p', round(d['ms_per_step'],3))" || tail -3 gpurun_out/pp.err
done; done
