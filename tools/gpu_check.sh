# usage: bash tools/gpu_check.sh [pytest -k expr] -- quick GPU validation + benches (no ncu)
set -x
K=${1:-}
if [ -n "$K" ]; then timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; else timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; fi
echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-2}; do timeout 600 python bench.py --config $c --no-cpu --e2e-steps 0 > gpurun_out/bench$c.json 2> gpurun_out/bench$c.err; echo bench$c=$?; tail -2 gpurun_out/bench$c.err; done
python tools/summarize_bench.py gpurun_out/bench*.json
