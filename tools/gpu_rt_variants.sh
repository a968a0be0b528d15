# usage: VARIANTS="-DX -DY" OPS="Rotate ShiftScaleRotate" bash tools/gpu_rt_variants.sh
# affine A/B (tools/affine_ab.py: rt vs pipe equality + timing) for the default
# build and each ALB_NVCC_FLAGS variant
OPS=${OPS:-Rotate ShiftScaleRotate}
bld() { ALB_NVCC_FLAGS="$1" python -c "from paper_1809_06839_b200 import build; build.build()"; }
for v in "" $VARIANTS; do
  bld "$v"; echo "== ${v:-default}"; python tools/affine_ab.py $OPS 2>&1 | grep -v Warn | grep -v "pipe  apply"
done
bld ""
