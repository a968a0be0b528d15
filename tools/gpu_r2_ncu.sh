# Round-2 evidence (part 2): ncu --set full captures (source-correlated) of
# the hot kernels, summarised ON THE BOX into CSV / text (raw metrics, per-line
# instruction counts of the top kernels) so the returned files stay small;
# the .ncu-rep files are deleted after summarising.
set -x
TAG=${TAG:-r2}
OPS=${OPS:-HorizontalFlip,Rotate,ShiftScaleRotate,Brightness,ShiftHSV,Grayscale,PadToSize512,Resize512,RandomSizedCrop64-512,Equalize,RandomCrop64}
python tools/profile_ops.py --ops $OPS --reps 1 > gpurun_out/plain_ops.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"k_(rowflip|rowgather|affine_rt|point|resample|eq_fused)" -c 14 -o /tmp/full_cfg2 python tools/profile_ops.py --ops $OPS --reps 1 > gpurun_out/ncu_full.log 2>&1; echo full=$?
python tools/profile_ops.py --ops cfg3:Rotate,cfg4,cfg5 --reps 1 > gpurun_out/plain_comp.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"k_(affine|resample|boxes|prep)" -c 10 -o /tmp/full_comp python tools/profile_ops.py --ops cfg3:Rotate,cfg4,cfg5 --reps 1 > gpurun_out/ncu_comp.log 2>&1; echo comp=$?
NOPS=${NOPS:-Rot90k1,Grid5,Elastic}
python tools/profile_ops.py --ops $NOPS --reps 1 > gpurun_out/plain_next.log 2>&1 && \
ncu -f --set full --clock-control none -k regex:"k_(d4|resample|elastic)" -c 3 -o /tmp/full_next python tools/profile_ops.py --ops $NOPS --reps 1 --n 500 > gpurun_out/ncu_next.log 2>&1; echo next=$?
for r in full_cfg2 full_comp full_next; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/${TAG}_${r}_raw.csv 2>/dev/null
done
python tools/ncu_lines.py /tmp/full_cfg2.ncu-rep k_affine_rt 40 > gpurun_out/${TAG}_lines_affine.txt 2>&1
python tools/ncu_lines.py /tmp/full_cfg2.ncu-rep k_resample_q4 40 > gpurun_out/${TAG}_lines_q4.txt 2>&1
python tools/ncu_lines.py /tmp/full_comp.ncu-rep k_resample 40 > gpurun_out/${TAG}_lines_cfg4.txt 2>&1
python tools/ncu_lines.py /tmp/full_cfg2.ncu-rep k_eq_fused 40 > gpurun_out/${TAG}_lines_eq.txt 2>&1
python tools/ncu_kstats.py /tmp/full_cfg2.ncu-rep k_affine_rt 288e6 > gpurun_out/${TAG}_kstats_affine.txt 2>&1
python tools/ncu_kstats.py /tmp/full_cfg2.ncu-rep k_resample_q4 > gpurun_out/${TAG}_kstats_q4.txt 2>&1
python tools/ncu_kstats.py /tmp/full_comp.ncu-rep k_affine_rt > gpurun_out/${TAG}_kstats_affine_cfg3.txt 2>&1
ls -la gpurun_out/
du -sh gpurun_out/
