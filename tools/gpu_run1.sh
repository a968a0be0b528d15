set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench=$?
for c in 3 4 5; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench$c.json 2> gpurun_out/bench$c.err; echo bench$c=$?; done
