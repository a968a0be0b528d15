# usage: OPS="Rotate" VARIANTS="-DA -DB" bash tools/gpu_ablate.sh
# timing of cfg2 transforms (tools/copy_probe.py) for the default build and
# each ablation build (ALB_NVCC_FLAGS variants; numbers from ablated builds are
# NOT valid outputs -- they bound how much time a removed part costs).
OPS=${OPS:-Rotate}
bld() { ALB_NVCC_FLAGS="$1" python -c "from paper_1809_06839_b200 import build; build.build()"; }
for v in "" $VARIANTS; do
  bld "$v"; echo "== ${v:-default}"; python tools/copy_probe.py $OPS 2>&1 | tail -n +2
done
bld ""
