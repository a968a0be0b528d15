# usage: FLAGS_B="-DX=1" bash tools/gpu_ab_cfg4.sh
# A/B of the cfg4 fused compose (bench.py --config 4) and cfg2 ShiftHSV
# (tools/copy_probe.py) between the default build and FLAGS_B, 3 alternating rounds.
bld() { ALB_NVCC_FLAGS="$1" python -c "from paper_1809_06839_b200 import build; build.build()"; }
bld "" && bld "$FLAGS_B"
for i in 1 2 3; do
  for v in "" "$FLAGS_B"; do
    bld "$v"; echo "== ${v:-default}"
    python tools/copy_probe.py ShiftHSV 2>&1 | tail -n +2
    timeout 300 python bench.py --config 4 --no-cpu --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4', d['ms_per_step'], 'ms', d['value'])"
  done
done
bld ""
