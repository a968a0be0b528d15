# tiles-per-CTA variants of the raw-tap affine kernel: cfg2 Rotate / SSR and cfg3 / cfg5 timings
bld() { ALB_NVCC_FLAGS="$1" python -c "from paper_1809_06839_b200 import build; build.build()"; }
for v in "" $VARIANTS; do
  bld "$v"; echo "== ${v:-default}"
  python tools/profile_ops.py --ops Rotate,ShiftScaleRotate,cfg3:Rotate,cfg3:ShiftScaleRotate,cfg5 --reps 3 --time 20 2>&1 | grep time
done
bld ""
