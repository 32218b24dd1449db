# Quick GPU check: parity tests matching $1 (pytest -k) and one bench line.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "${1:-compress}" 2>&1 | tail -25
timeout 600 python bench.py > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; cat gpurun_out/bench_quick.json; tail -5 gpurun_out/bench_quick.err
