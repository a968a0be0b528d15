# usage: OPS="Resize512 RandomSizedCrop64-512" FLAGS_B="-DX=1" bash tools/gpu_ab.sh
# A/B timing of cfg2 transforms (tools/copy_probe.py) between the default build and
# a build with extra nvcc flags (ALB_NVCC_FLAGS), 3 alternating rounds (each
# switch relinks libalb_b200.so from the cached object set of that flag set).
OPS=${OPS:-Resize512}
bld() { ALB_NVCC_FLAGS="$1" python -c "from paper_1809_06839_b200 import build; build.build()"; }
bld "" && bld "$FLAGS_B"
for i in 1 2 3; do
  bld ""; echo "== A"; python tools/copy_probe.py $OPS 2>&1 | tail -n +2
  bld "$FLAGS_B"; echo "== B $FLAGS_B"; python tools/copy_probe.py $OPS 2>&1 | tail -n +2
done
bld ""
