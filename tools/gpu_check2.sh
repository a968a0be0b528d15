# usage: bash tools/gpu_check2.sh [pytest -k expr]
# GPU tests (optionally filtered), smoke, and the default bench line (cfg2 + composed configs).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
K=${1:-}
if [ -n "$K" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; else timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; fi
echo pytest=$?
grep -E "FAILED|Error|passed|failed" gpurun_out/pytest_gpu.log | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -3 gpurun_out/smoke.log
if [ -z "${NOBENCH:-}" ]; then
timeout 900 python bench.py ${BENCH_ARGS:---no-cpu} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; tail -3 gpurun_out/bench.err
python tools/summarize_bench.py gpurun_out/bench.json
fi
