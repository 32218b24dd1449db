mkdir -p gpurun_out
for cfg in "0 0" "0 1" "24 0" "48 0" "48 1" "74 1"; do set -- $cfg
timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 3 --overlap-bwd 4096 --bwd-carveout $1 --lsp-priority $2 > gpurun_out/ovl.json 2> gpurun_out/ovl.err; python -c "
import json;d=json.load(open('gpurun_out/ovl.json'))['overlap'];print('carve=$1 prio=$2', {k:(round(v,2) if isinstance(v,float) else v) for k,v in d.items() if k not in ('note',)})" || tail -3 gpurun_out/ovl.err
done
