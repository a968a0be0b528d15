#!/usr/bin/env python
"""Benchmark of the B200 augmentation hot path (BASELINE.json metric:
"images/sec per transform and composed pipeline; % of B200 HBM roofline").

One STEP = every transform of the cfg2 menu (BASELINE.json configs[1]: 16
single transforms, each its own alb_apply) over the 2000-image ragged corpus
already resident in HBM.  `value` = images that went through the whole menu
per second, summed over ranks (weak scaling: each rank owns its own 2000
images, global indices rank*2000 + i; no collective on the data path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2|3|4|5]

Under torchrun every rank runs its shard; rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import configs as C  # noqa: E402
from synth import gen  # noqa: E402

METRIC = "images/sec per transform and composed pipeline; % of B200 HBM roofline"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ----------------------------------------------------------------- workloads

def workload(cfg, rank):
    """(name, op menu {label: specs}, sizes, extra) for a config."""
    if cfg == 2:
        n = C.CONFIGS[2]["n"]
        sizes = gen.cfg2_sizes(n, first_image_index=rank * n)
        return ("cfg2: 2000 ragged RGB images W in [400,500], H = 0.75 W (R24), gradient+noise; "
                "16 single transforms, p = 1"), dict(C.CFG2_MENU), sizes, {}
    if cfg == 3:
        n = C.CONFIGS[3]["n"]
        return ("cfg3: 256 RGB 512x512 + uint8 mask; Rotate(+-90), SSR; bilinear, reflect_101",
                dict(C.CFG3_OPS), [(512, 512)] * n, {"masks": True})
    if cfg == 4:
        n = C.CONFIGS[4]["n"]
        return ("cfg4: 1024 RGB 500x375 per GPU; RSC(64-375)->Resize224->HFlip(.5)->ShiftHSV->BC->"
                "Normalize to fp32 NCHW", {"cfg4_compose": C.CFG4_OPS}, [(375, 500)] * n, {})
    if cfg == 5:
        n = C.CONFIGS[5]["n"]
        return ("cfg5: 512 RGB 1024x1024 per GPU + mask + 0-50 boxes; SSR+RandomCrop512+HFlip(.5), "
                "min-visibility 0.3", {"cfg5_compose": C.CFG5_OPS}, [(1024, 1024)] * n,
                {"masks": True, "boxes": True})
    raise SystemExit("unknown config %d" % cfg)


def alg_bytes(label, specs, sizes, prm=None):
    """Algorithmic bytes (read + write) of one apply over the batch (DESIGN.md
    measurement section).  prm: device-drawn params (RSC side)."""
    tot = 0
    last = specs[-1]["kind"]
    for i, (h, w) in enumerate(sizes):
        inb = h * w * 3
        kind = specs[0]["kind"]
        if label == "cfg4_compose":
            side = int(prm[i, 0, 0])
            tot += side * side * 3 + 3 * 224 * 224 * 4
        elif label == "cfg5_compose":
            s = float(prm[i, 0, 2])
            foot = min(h * w, int(512 * 512 / (s * s)))
            tot += foot * 4 + 512 * 512 * 4
        elif kind == "RandomCrop":
            ow, oh = specs[0]["size"]
            tot += 2 * ow * oh * 3
        elif kind in ("PadToSize", "Resize"):
            ow, oh = specs[0]["size"]
            tot += inb + ow * oh * 3
        elif kind == "RandomSizedCrop":
            side = int(prm[i, 0, 0])
            ow, oh = specs[0]["size"]
            tot += side * side * 3 + ow * oh * 3
        else:
            tot += 2 * inb
    del last
    return tot


class Clocks(threading.Thread):
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        super().__init__(daemon=True)
        self.index = index
        self.rows = []
        self.proc = None

    def run(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            for line in self.proc.stdout:
                self.rows.append([t.strip() for t in line.split(",")])
        except Exception:
            pass

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 2 + k and r[2 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ------------------------------------------------------------ oracle timing

def oracle_menu_rate(menu, sizes, n_img, seed, threads, first=0, batch=None):
    """Oracle (as it stands) over the first n_img images of the workload: returns
    (images through the whole menu per second, seconds).  `batch` (if given)
    supplies the images already generated for the GPU run."""
    from oracle import albref as A
    if batch is None:
        batch = gen.gen_images(sizes[:n_img], seed=0, first_image_index=first, device="cpu")
    imgs = [batch.image(i) for i in range(n_img)]
    t0 = time.perf_counter()
    for label, specs in menu.items():
        A.apply_batch(specs, seed, first, imgs, threads=threads)
    dt = time.perf_counter() - t0
    return n_img / dt, dt


# -------------------------------------------------------------------- main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    peak, peak_src = peaks()

    if args.impl == "reference":
        return run_reference(args, world, rank)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)

    from paper_1809_06839_b200 import Layout, Pipeline, Plan, build
    build.build()

    name, menu, sizes, extra = workload(args.config, rank)
    n = len(sizes)
    first = rank * n
    batch = gen.gen_images(sizes, seed=0, first_image_index=first, device=dev)
    masks = boxes = None
    if extra.get("masks"):
        bx, lb, cnt, masks = gen.gen_boxes(sizes, seed=0, first_image_index=first,
                                           with_mask=True)
        masks = masks.to(dev)
        if extra.get("boxes"):
            boxes = [torch.from_numpy(bx).to(dev), torch.from_numpy(lb).to(dev),
                     torch.from_numpy(cnt).to(dev)]
    in_l = Layout(batch.desc, 3)
    m_l = Layout(masks.desc, 1) if masks is not None else None

    plans = {}
    for label, specs in menu.items():
        pipe = Pipeline(specs)
        osz = [pipe.output_shape(h, w) for h, w in sizes]
        ends_norm = specs[-1]["kind"] == "Normalize"
        ob = None if ends_norm else gen.empty_batch(osz, 3, dev)
        nchw = (torch.empty((n, 3) + tuple(osz[0]), dtype=torch.float32, device=dev)
                if ends_norm else None)
        ol = None if ob is None else Layout(ob.desc, 3)
        mo = mol = None
        if masks is not None:
            mo = gen.empty_batch(osz, 1, dev)
            mol = Layout(mo.desc, 1)
        bo = None
        if boxes is not None:
            bo = [torch.empty_like(boxes[0]), torch.empty_like(boxes[1]), torch.empty_like(boxes[2])]
        plan = Plan(pipe, in_l, ol, m_l, mol, C.CFG5_MAX_BOXES if boxes is not None else 0,
                    C.CFG5_MIN_VISIBILITY if boxes is not None else 0.0)
        plans[label] = dict(pipe=pipe, plan=plan, out=ob, nchw=nchw, mo=mo, bo=bo, ol=ol, mol=mol,
                            ws=plan.workspace(dev), specs=specs)

    stream = torch.cuda.current_stream(dev)

    def apply_one(label, seed):
        P = plans[label]
        bi = boxes if boxes is not None else [None] * 3
        bo = P["bo"] if P["bo"] is not None else [None] * 3
        P["plan"].apply(seed, first, batch.buf, None if P["out"] is None else P["out"].buf,
                        P["nchw"], None if masks is None else masks.buf,
                        None if P["mo"] is None else P["mo"].buf, bi[0], bi[1], bi[2],
                        bo[0], bo[1], bo[2], workspace=P["ws"], stream=stream)

    labels = list(menu)
    for s in range(args.warmup):
        for label in labels:
            apply_one(label, args.seed + 1000 + s)
    torch.cuda.synchronize()

    # algorithmic bytes per step for each op (params drawn by the device sampler)
    hw = np.array(sizes, np.int32)
    seeds = [args.seed + s for s in range(args.steps)]
    bytes_per = {label: 0 for label in labels}
    for s in seeds:
        for label in labels:
            prm = None
            if menu[label][0]["kind"] in ("RandomSizedCrop", "ShiftScaleRotate"):
                prm, _ = plans[label]["pipe"].sample_params(s, first, hw)
            bytes_per[label] += alg_bytes(label, menu[label], sizes, prm)

    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.5)
    ev = {label: [] for label in labels}
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for s in seeds:
        for label in labels:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            apply_one(label, s)
            e1.record(stream)
            ev[label].append((e0, e1))
    t_end.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks.stop()
    elapsed = t_start.elapsed_time(t_end) / 1e3
    op_time = {label: sum(a.elapsed_time(b) for a, b in ev[label]) / 1e3 for label in labels}
    t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_max = float(t.item())

    launches = args.steps * sum(P["plan"].num_launches for P in plans.values())
    per = {}
    for label in labels:
        gbs = bytes_per[label] / op_time[label] / 1e9
        per[label] = {"images_per_s": round(world * n * args.steps / op_time[label], 1),
                      "ms_per_apply": round(op_time[label] / args.steps * 1e3, 4),
                      "alg_GBps": round(gbs, 1), "frac_of_peak": round(gbs / peak, 4)}
    dom = max(labels, key=lambda l: op_time[l])
    dom_gbs = bytes_per[dom] / op_time[dom] / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("cfg%d" % args.config, {}).get(dom)

    # ---------------------------------------------------------------- e2e
    e2e = None
    if args.e2e_steps > 0 and "cfg2" in name:
        host_in = batch.buf.cpu().pin_memory()
        dev_in = torch.empty_like(batch.buf)
        hosts = {}
        for label in labels:
            P = plans[label]
            dout = P["out"].buf if P["out"] is not None else P["nchw"]
            hosts[label] = (torch.empty(dout.shape, dtype=dout.dtype).pin_memory(),
                            torch.empty_like(dout))
        for label in labels:  # warm
            plans[label]["plan"].apply_host(args.seed, first, host_in, dev_in, hosts[label][0],
                                            hosts[label][1], plans[label]["ws"], stream)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(args.e2e_steps):
            for label in labels:
                plans[label]["plan"].apply_host(args.seed + s, first, host_in, dev_in,
                                                hosts[label][0], hosts[label][1],
                                                plans[label]["ws"], stream)
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=dev)
        if dist:
            dist.barrier()
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        h2d = len(labels) * host_in.numel()
        d2h = sum(h[0].numel() * h[0].element_size() for h in hosts.values())
        e2e = {"value": round(world * n * args.e2e_steps / float(te.item()), 2),
               "unit": "images/s (full 16-transform menu, pinned host in -> HBM -> host out)",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # ------------------------------------------------------- cpu baseline
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        n_img = 2000 if args.config == 2 else 16  # ~10 s of host work on the GPU box
        host = gen.Batch(batch.buf.cpu(), batch.desc, 3)
        rate, dt = oracle_menu_rate(menu, sizes, n_img, args.seed, threads, first, host)
        cpu = {"value": round(rate, 3), "unit": "images/s (whole menu)", "cores": threads,
               "kind": "oracle",
               "sample": "first %d images of the same workload, every transform of the menu, "
                         "oracle/libalbref.so (plain C fp64) on %d host threads, %.1f s" % (
                             n_img, threads, dt)}

    if rank == 0:
        out = {
            "metric": METRIC,
            "value": round(world * n * args.steps / elapsed_max, 2),
            "unit": "images/s (each image through all %d transforms of the menu)" % len(labels)
            if "cfg2" in name else "images/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(elapsed_max / args.steps * 1e3, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic (seeded gradient+noise, synth/gen.py)",
            "config": {"workload": name, "images_per_gpu": n, "global_batch": n * world,
                       "parallelism": "dp%d (independent shards, no collective)" % world,
                       "l2": "inputs larger than L2 (%.0f MB corpus per GPU), seed advances per step"
                             % (batch.buf.numel() / 1e6)},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(dom_gbs, 1),
                         "peak": peak, "unit": "GB/s", "frac": round(dom_gbs / peak, 4),
                         "traffic": traffic, "peak_source": peak_src,
                         "note": "achieved = algorithmic bytes of the dominant transform / its "
                                 "apply duration (CUDA events on the launch stream; includes the "
                                 "K0 param/LUT launch)"},
            "per_transform": per,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


def run_reference(args, world, rank):
    """--impl reference: the oracle as it stands, on the host cores, bounded."""
    if rank != 0:
        return
    name, menu, sizes, _ = workload(args.config, 0)
    threads = os.cpu_count() or 1
    n_img = 256 if args.config == 2 else 4
    for s in range(args.warmup):
        oracle_menu_rate(menu, sizes, 2, args.seed + s, threads)
    t = 0.0
    for s in range(args.steps):
        _, dt = oracle_menu_rate(menu, sizes, n_img, args.seed + s, threads)
        t += dt
    val = n_img * args.steps / t
    unit = "images/s (each image through all %d transforms of the menu)" % len(menu)
    out = {"impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": unit,
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(t / args.steps * 1e3, 2), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": name, "images_per_step": n_img},
           "cpu_baseline": {"value": round(val, 3), "unit": unit, "cores": threads,
                            "kind": "oracle",
                            "sample": "each step = first %d images of the workload through the "
                                      "whole menu, plain C oracle" % n_img},
           "e2e": {"value": round(val, 3), "unit": unit, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
