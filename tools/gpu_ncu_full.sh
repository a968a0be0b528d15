# Round evidence (part 2): one ncu --set full capture of each distinct hot
# kernel of the cfg2 menu (one transform per kernel family), source-correlated.
OPS=${OPS:-HorizontalFlip,Rotate,ShiftScaleRotate,Brightness,ShiftHSV,Grayscale,PadToSize512,Resize512,Equalize}
python tools/profile_ops.py --ops $OPS --reps 1 > gpurun_out/plain_ops.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(rowflip|rowgather|affine_pipe|point|resample|eq_hist)" -c 12 -o gpurun_out/full_cfg2 python tools/profile_ops.py --ops $OPS --reps 1 > gpurun_out/ncu_full.log 2>&1; echo full=$?
tail -3 gpurun_out/ncu_full.log
ls -la gpurun_out/
# next-row kernels (§8(f)): Rotate90 (k_d4), GridDistortion (k_resample_sep), ElasticTransform (k_elastic)
NOPS=${NOPS:-Rot90k1,Grid5,Elastic}
python tools/profile_ops.py --ops $NOPS --reps 1 > gpurun_out/plain_next.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_(d4|resample|elastic)" -c 3 -o gpurun_out/full_next python tools/profile_ops.py --ops $NOPS --reps 1 --n 500 > gpurun_out/ncu_next.log 2>&1; echo next=$?
ls -la gpurun_out/*.ncu-rep
