# Round-2 evidence on one B200 (part 1, small outputs): GPU tests, smoke, the
# default bench line (cfg2 + composed configs), the reference arm, the ncu
# launch list of the bench command, the decode -> cfg4 end-to-end line.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
CMD="python bench.py --config 2 --steps 2 --warmup 3 --no-cpu --e2e-steps 0"
$CMD > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 800 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo launches=$?
timeout 600 python tools/decode_probe.py --n 2000 --reps 5 --json gpurun_out/f3_e2e.json > gpurun_out/decode.log 2>&1; echo decode=$?
ls -la gpurun_out/
