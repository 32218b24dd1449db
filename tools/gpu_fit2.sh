# Fit engine on fast fp64 gathers: fit / parity / conformance tests, then C3-shape timing.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fit.py tests/test_gpu_parity.py tests/test_gpu_conformance.py -m gpu -x -q > gpurun_out/pytest_fit.log 2>&1; tail -15 gpurun_out/pytest_fit.log
timeout 900 python tools/time_fit.py 2048 5504 1024 4 9 > gpurun_out/time_fit.json 2>&1; tail -c 1200 gpurun_out/time_fit.json
