# Round-2 evidence on one B200: GPU tests, smoke, the default bench line (cfg2 +
# composed configs) and the reference arm, the ncu launch list of the bench
# command, full ncu captures of the hot kernels (cfg2 families + composed
# configs' kernels), and the decode -> cfg4 end-to-end line.
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
OPS=${OPS:-HorizontalFlip,Rotate,ShiftScaleRotate,Brightness,ShiftHSV,Grayscale,PadToSize512,Resize512,RandomSizedCrop64-512,Equalize,RandomCrop64}
python tools/profile_ops.py --ops $OPS --reps 1 > gpurun_out/plain_ops.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(rowflip|rowgather|affine_pipe|point|resample|eq_fused)" -c 14 -o gpurun_out/full_cfg2 python tools/profile_ops.py --ops $OPS --reps 1 > gpurun_out/ncu_full.log 2>&1; echo full=$?
python tools/profile_ops.py --ops cfg3:Rotate,cfg4,cfg5 --reps 1 > gpurun_out/plain_comp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(affine|resample|boxes|prep)" -c 10 -o gpurun_out/full_comp python tools/profile_ops.py --ops cfg3:Rotate,cfg4,cfg5 --reps 1 > gpurun_out/ncu_comp.log 2>&1; echo comp=$?
timeout 600 python tools/decode_probe.py --n 2000 --reps 5 --json gpurun_out/f3_e2e.json > gpurun_out/decode.log 2>&1; echo decode=$?
ls -la gpurun_out/
