#!/usr/bin/env python
"""Benchmark of the B200 augmentation hot path (BASELINE.json metric:
"images/sec per transform and composed pipeline; % of B200 HBM roofline").

One STEP = every transform of the cfg2 menu (BASELINE.json configs[1]: 16
single transforms, each its own alb_apply) over the 2000-image ragged corpus
already resident in HBM.  `value` = images that went through the whole menu
per second, summed over ranks (weak scaling: each rank owns its own 2000
images, global indices rank*2000 + i; no collective on the data path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 0|2|3|4|5]

The default run (--config 0) measures the cfg2 menu as the headline line and
the composed configs (cfg3 warps with masks, cfg4 fused Compose -> fp32 NCHW,
cfg5 co-transform with masks and boxes) into its "composed" object, each
with its own images/s, roofline and end-to-end number.  Under torchrun every
rank runs its shard; rank 0 prints ONE JSON line.
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


def alg_bytes(label, specs, sizes, prm=None, masks=False, boxes=False):
    """Algorithmic bytes (read + write) of one apply over the batch (DESIGN.md
    measurement section).  prm: device-drawn params (RSC side)."""
    tot = 0
    cpp = 4 if masks else 3  # bytes per pixel moved: RGB (+ the uint8 label)
    for i, (h, w) in enumerate(sizes):
        inb = h * w * cpp
        kind = specs[0]["kind"]
        if boxes:
            tot += 2 * 16 * C.CFG5_MAX_BOXES + 2 * 4 * C.CFG5_MAX_BOXES + 8  # xyxy + labels + count, in and out
        if label == "cfg4_compose":
            side = int(prm[i, 0, 0])
            tot += side * side * 3 + 3 * 224 * 224 * 4
        elif label == "cfg5_compose":
            s = float(prm[i, 0, 2])
            foot = min(h * w, int(512 * 512 / (s * s)))
            tot += foot * 4 + 512 * 512 * 4
        elif kind == "RandomCrop":
            ow, oh = specs[0]["size"]
            tot += 2 * ow * oh * cpp
        elif kind in ("PadToSize", "Resize"):
            ow, oh = specs[0]["size"]
            tot += inb + ow * oh * cpp
        elif kind == "RandomSizedCrop":
            side = int(prm[i, 0, 0])
            ow, oh = specs[0]["size"]
            tot += side * side * cpp + ow * oh * cpp
        else:
            tot += 2 * inb
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

ALL_CONFIGS = (2, 3, 4, 5)


def config_dict(cfg, name, sizes, world):
    """The `config` object of a line (identical in both arms for one config)."""
    n = len(sizes)
    _, total = gen.layout(sizes, 3)
    return {"workload": name, "images_per_gpu": n, "global_batch": n * world,
            "parallelism": "dp%d (independent shards, no collective)" % world,
            "l2": "inputs larger than L2 (%.0f MB of images per GPU), seed advances per step"
                  % (total / 1e6)}


def unit_of(cfg, menu):
    if cfg == 2:
        return "images/s (each image through all %d transforms of the menu)" % len(menu)
    return "images/s (each image through the %s)" % (
        "composed pipeline" if len(menu) == 1 else "%d transforms of the config" % len(menu))


class Workload:
    """Inputs (resident in HBM), plans, outputs and workspaces of one config."""

    def __init__(self, cfg, rank, dev):
        from paper_1809_06839_b200 import Layout, Pipeline, Plan
        self.cfg = cfg
        self.name, self.menu, self.sizes, self.extra = workload(cfg, rank)
        self.n = n = len(self.sizes)
        self.first = rank * n
        self.dev = dev
        self.batch = gen.gen_images(self.sizes, seed=0, first_image_index=self.first, device=dev)
        self.masks = self.boxes = None
        if self.extra.get("masks"):
            bx, lb, cnt, masks = gen.gen_boxes(self.sizes, seed=0, first_image_index=self.first,
                                               with_mask=True)
            self.masks = masks.to(dev)
            if self.extra.get("boxes"):
                self.boxes = [torch.from_numpy(bx).to(dev), torch.from_numpy(lb).to(dev),
                              torch.from_numpy(cnt).to(dev)]
        in_l = Layout(self.batch.desc, 3)
        m_l = Layout(self.masks.desc, 1) if self.masks is not None else None
        self.plans = {}
        for label, specs in self.menu.items():
            pipe = Pipeline(specs)
            osz = [pipe.output_shape(h, w) for h, w in self.sizes]
            ends_norm = specs[-1]["kind"] == "Normalize"
            ob = None if ends_norm else gen.empty_batch(osz, 3, dev)
            nchw = (torch.empty((n, 3) + tuple(osz[0]), dtype=torch.float32, device=dev)
                    if ends_norm else None)
            ol = None if ob is None else Layout(ob.desc, 3)
            mo = mol = None
            if self.masks is not None:
                mo = gen.empty_batch(osz, 1, dev)
                mol = Layout(mo.desc, 1)
            bo = None
            if self.boxes is not None:
                bo = [torch.empty_like(t) for t in self.boxes]
            mb = C.CFG5_MAX_BOXES if self.boxes is not None else 0
            plan = Plan(pipe, in_l, ol, m_l, mol, mb,
                        C.CFG5_MIN_VISIBILITY if self.boxes is not None else 0.0)
            self.plans[label] = dict(pipe=pipe, plan=plan, out=ob, nchw=nchw, mo=mo, bo=bo, ol=ol,
                                     mol=mol, ws=plan.workspace(dev), specs=specs)
        self.layouts = (in_l, m_l)

    def apply(self, label, seed, stream, img_in=None, mask_in=None, boxes_in=None, res=None):
        """res: optional (out buffer, nchw, mask out buffer, box outs, workspace)
        replacing the plan's own (a second in-flight copy, bench e2e)."""
        P = self.plans[label]
        out, nchw, mo, bo, ws = res or (None if P["out"] is None else P["out"].buf, P["nchw"],
                                        None if P["mo"] is None else P["mo"].buf, P["bo"], P["ws"])
        bi = boxes_in or self.boxes or [None] * 3
        bo = bo or [None] * 3
        masks_in = mask_in if mask_in is not None else (None if self.masks is None else self.masks.buf)
        P["plan"].apply(seed, self.first, self.batch.buf if img_in is None else img_in, out, nchw, masks_in,
                        mo, bi[0], bi[1], bi[2], bo[0], bo[1], bo[2], workspace=ws, stream=stream)

    def alg_bytes(self, seeds):
        hw = np.array(self.sizes, np.int32)
        per = {label: 0 for label in self.menu}
        for s in seeds:
            for label, specs in self.menu.items():
                prm = None
                if specs[0]["kind"] in ("RandomSizedCrop", "ShiftScaleRotate"):
                    prm, _ = self.plans[label]["pipe"].sample_params(s, self.first, hw)
                per[label] += alg_bytes(label, specs, self.sizes, prm,
                                        masks=self.masks is not None,
                                        boxes=self.boxes is not None)
        return per

    def launches(self):
        return sum(P["plan"].num_launches for P in self.plans.values())


def timed_steps(W, seeds, stream, dist, dev):
    """Time len(seeds) steps (every transform of the menu once per step) between
    a barrier + synchronize on both sides; per-apply CUDA events on the launch
    stream.  Returns (max-over-ranks elapsed s, {label: [s per apply]}, [s per step])."""
    labels = list(W.menu)
    ev = {label: [] for label in labels}
    bounds = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for s in seeds:
        eb = torch.cuda.Event(enable_timing=True)
        eb.record(stream)
        bounds.append(eb)
        for label in labels:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            W.apply(label, s, stream)
            e1.record(stream)
            ev[label].append((e0, e1))
    t1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t = torch.tensor([t0.elapsed_time(t1) / 1e3], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    bounds.append(t1)
    steps = [a.elapsed_time(b) / 1e3 for a, b in zip(bounds[:-1], bounds[1:])]
    return float(t.item()), {l: [a.elapsed_time(b) / 1e3 for a, b in ev[l]] for l in labels}, steps


def graph_times(W, seeds, dev):
    """Per transform: the step's applies (one per seed) captured into CUDA
    graphs before timing, then replayed back to back between two events on a
    side stream: the kernels without per-launch host overhead or gaps.
    Returns {label: seconds per apply}."""
    s = torch.cuda.Stream(dev)
    out = {}
    for label in W.menu:
        graphs = []
        for seed in seeds:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                W.apply(label, seed, s)
            graphs.append(g)
        for g in graphs:  # warm
            g.replay()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for g in graphs:
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        out[label] = e0.elapsed_time(e1) / 1e3 / len(graphs)
        del graphs
    return out


def e2e_run(W, args, stream, dist, dev, world):
    """The same metric end to end through the public API with HOST buffers:
    every step copies its inputs from pinned host memory and its results back,
    inside the timed region.  Unmasked plans use alb_apply_host (chunked,
    copies overlapping the kernels); masked / boxed plans copy images, masks and
    boxes in with torch and call alb_apply.  Two applies are in flight on two
    streams (transform i of the menu on stream i % 2; a one-transform menu
    alternates steps, with a second set of device buffers and workspace), so
    one apply's result copy overlaps the next one's input copy: the host link
    carries both directions at once."""
    labels = list(W.menu)
    streams = [stream, torch.cuda.Stream(dev)]
    by_step = len(labels) == 1
    host_in = W.batch.buf.cpu().pin_memory()
    dev_in = [torch.empty_like(W.batch.buf) for _ in streams]
    hm = dm = hb = db = None
    if W.masks is not None:
        hm = W.masks.buf.cpu().pin_memory()
        dm = [torch.empty_like(W.masks.buf) for _ in streams]
    if W.boxes is not None:
        hb = [t.cpu().pin_memory() for t in W.boxes]
        db = [[torch.empty_like(t) for t in W.boxes] for _ in streams]
    # device results per (transform, stream): the plan's own on its first
    # stream, a twin set (and workspace) on the second when steps alternate
    res = {}
    home = {label: 0 if by_step else li % 2 for li, label in enumerate(labels)}
    for label in labels:
        P = W.plans[label]
        res[(label, home[label])] = (None if P["out"] is None else P["out"].buf, P["nchw"],
                                     None if P["mo"] is None else P["mo"].buf, P["bo"], P["ws"])
        if by_step:
            o, n, m, b, w = res[(label, 0)]
            res[(label, 1)] = tuple(None if t is None else ([torch.empty_like(x) for x in t] if isinstance(t, list)
                                                            else torch.empty_like(t)) for t in (o, n, m, b, w))
    # one pinned host arena per stream for every transform's results (each
    # D2H lands at its arena's start; the bytes read back per step are still
    # every result): ~3 corpora of pinned memory per rank
    arena_bytes = 0
    for label in labels:
        o, n, m, b, _ = res[(label, home[label])]
        arena_bytes = max(arena_bytes, sum(t.numel() * t.element_size() for t in [o if o is not None else n] +
                                           ([m] if m is not None else []) + (b or [])))
    arenas = [torch.empty(arena_bytes + 256 * 8, dtype=torch.uint8).pin_memory() for _ in streams]

    def host_views(j, outs):
        views, pos = [], 0
        for o in outs:
            nb = o.numel() * o.element_size()
            views.append((arenas[j][pos:pos + nb].view(o.dtype).view(o.shape), o))
            pos = (pos + nb + 255) // 256 * 256
        return views

    hosts = {}
    for (label, j), (o, n, m, b, w) in res.items():
        hosts[(label, j)] = host_views(j, [o if o is not None else n] + ([m] if m is not None else []) + (b or []))

    def step(seed, si):
        for li, label in enumerate(labels):
            j = si % 2 if by_step else home[label]
            st = streams[j]
            P = W.plans[label]
            r = res[(label, j)]
            if hm is None and hb is None:
                (ho, do), = hosts[(label, j)]
                P["plan"].apply_host(seed, W.first, host_in, dev_in[j], ho, do, r[4], st)
                continue
            with torch.cuda.stream(st):
                dev_in[j].copy_(host_in, non_blocking=True)
                if hm is not None:
                    dm[j].copy_(hm, non_blocking=True)
                if hb is not None:
                    for d, h in zip(db[j], hb):
                        d.copy_(h, non_blocking=True)
                W.apply(label, seed, st, img_in=dev_in[j], mask_in=None if dm is None else dm[j],
                        boxes_in=None if db is None else db[j], res=r)
                for ho, do in hosts[(label, j)]:
                    ho.copy_(do, non_blocking=True)

    step(args.seed, 0)  # warm
    step(args.seed, 1)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    streams[1].wait_event(e0)
    for s in range(args.e2e_steps):
        step(args.seed + s, s)
    j1 = torch.cuda.Event()
    j1.record(streams[1])
    stream.wait_event(j1)
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=dev)
    if dist:
        dist.barrier()
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    in_bytes = host_in.numel() + (hm.numel() if hm is not None else 0) + \
        (sum(t.numel() * t.element_size() for t in hb) if hb is not None else 0)
    h2d = len(labels) * in_bytes
    d2h = sum(h.numel() * h.element_size() for (label, j), v in hosts.items() if j == home[label] for h, _ in v)
    return {"value": round(world * W.n * args.e2e_steps / float(te.item()), 2),
            "unit": unit_of(W.cfg, W.menu),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "path": ("alb_apply_host (pinned host in -> HBM -> kernels -> pinned host out, 16 image chunks, "
                     "copies overlap kernels)" if hm is None and hb is None else
                     "pinned host images/masks/boxes -> HBM (torch copies), alb_apply, results -> pinned host")
                    + "; two applies in flight on two streams"}


def measure(cfg, args, dev, rank, world, dist, peak, peak_src, local):
    """One config: warm up, time K steps, per-transform numbers, roofline, e2e."""
    W = Workload(cfg, rank, dev)
    stream = torch.cuda.current_stream(dev)
    labels = list(W.menu)
    # the headline config times exactly K steps; a composed config (a ~1 ms
    # step) times at least 20 (>= 20 passes or >= 200 ms)
    steps = args.steps if cfg == (ALL_CONFIGS[0] if args.config == 0 else args.config) else max(args.steps, 20)
    seeds = [args.seed + s for s in range(steps)]
    bytes_per = W.alg_bytes(seeds)  # host work, before the GPU is warmed

    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.5)
    # warm-up right before the timed steps (after the sampler started), so
    # the first timed step does not run on clocks that dropped while idle
    for s in range(args.warmup):
        for label in labels:
            W.apply(label, args.seed + 1000 + s, stream)
    torch.cuda.synchronize()
    elapsed, op_times, step_times = timed_steps(W, seeds, stream, dist, dev)
    clocks.stop()
    per = {}
    for label in labels:
        ts = op_times[label]
        tot = sum(ts)
        gbs = bytes_per[label] / tot / 1e9
        per[label] = {"images_per_s": round(world * W.n * len(ts) / tot, 1),
                      "ms_per_apply": round(tot / len(ts) * 1e3, 4),
                      "ms_median": round(statistics.median(ts) * 1e3, 4),
                      "alg_GBps": round(gbs, 1), "frac_of_peak": round(gbs / peak, 4)}
    if args.graph:  # each apply replayed from a CUDA graph (launch-bound ops)
        g_times = graph_times(W, seeds, dev)
        for label in labels:
            tg = g_times[label]
            per[label]["ms_per_apply_graph"] = round(tg * 1e3, 4)
            per[label]["frac_of_peak_graph"] = round(bytes_per[label] / len(seeds) / tg / 1e9 / peak, 4)
    dom = max(labels, key=lambda l: sum(op_times[l]))
    dom_gbs = bytes_per[dom] / sum(op_times[dom]) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("cfg%d" % cfg, {}).get(dom)
    e2e = e2e_run(W, args, stream, dist, dev, world) if args.e2e_steps > 0 else None
    res = {
        "value": round(world * W.n * steps / elapsed, 2),
        "steps": steps,
        "unit": unit_of(cfg, W.menu),
        "ms_per_step": round(elapsed / steps * 1e3, 4),
        "config": config_dict(cfg, W.name, W.sizes, world),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(dom_gbs, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(dom_gbs / peak, 4),
                     "traffic": traffic, "peak_source": peak_src,
                     "note": "achieved = algorithmic bytes of the dominant transform / its "
                             "apply duration (CUDA events on the launch stream around the "
                             "whole alb_apply, K0 parameter launch included)"},
        "per_transform": per,
        "trials": trials_of(step_times, world * W.n),
        "e2e": e2e,
        "gpu_launches": steps * W.launches(),
        "clocks": clocks.summary(),
    }
    return W, res


def trials_of(step_times, images_per_step, n=5):
    """the K timed steps as n consecutive trials (this rank's
    CUDA events between step boundaries); images/s of each and the median."""
    if len(step_times) < n:
        n = len(step_times)
    if n == 0:
        return None
    k = len(step_times) // n
    ips = [images_per_step * k / sum(step_times[i * k:(i + 1) * k]) for i in range(n)]
    return {"n": n, "steps_each": k, "images_per_s": [round(v, 1) for v in ips],
            "median": round(statistics.median(ips), 1)}


def cpu_baseline(W, args):
    """The oracle as it stands, on the host cores: all 2000 cfg2 images through
    the menu on every core, plus a single-threaded 32-image subset."""
    threads = os.cpu_count() or 1
    n_img = min(W.n, 2000 if W.cfg == 2 else 16)
    host = gen.Batch(W.batch.buf.cpu(), W.batch.desc, 3)
    rate, dt = oracle_menu_rate(W.menu, W.sizes, n_img, args.seed, threads, W.first, host)
    n1 = min(n_img, 32 if W.cfg == 2 else 2)
    rate1, dt1 = oracle_menu_rate(W.menu, W.sizes, n1, args.seed, 1, W.first, host)
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"value": round(rate, 3), "unit": unit_of(W.cfg, W.menu), "cores": threads,
            "kind": "oracle", "cpu_model": model,
            "single_thread": {"value": round(rate1, 3), "images": n1, "seconds": round(dt1, 2)},
            "sample": "first %d images of the same workload, every transform of the menu, "
                      "oracle/libalbref.so (plain C fp64) on %d host threads, %.1f s" % (
                          n_img, threads, dt)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=0,
                    help="0 (default): cfg2 menu as the headline + cfg3/4/5 composed configs")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="skip the per-transform CUDA-graph replay timing")
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

    from paper_1809_06839_b200 import build
    build.build()

    cfgs = ALL_CONFIGS if args.config == 0 else (args.config,)
    head = None
    composed = {}
    cpu = None
    for cfg in cfgs:
        W, res = measure(cfg, args, dev, rank, world, dist, peak, peak_src, local)
        if head is None:
            head = res
            if rank == 0 and world == 1 and not args.no_cpu:
                cpu = cpu_baseline(W, args)
        else:
            composed["cfg%d" % cfg] = res
        del W
        torch.cuda.empty_cache()
        if hasattr(torch._C, "_host_emptyCache"):  # return this config's pinned host buffers
            torch._C._host_emptyCache()

    if rank == 0:
        out = {"metric": METRIC, "value": head["value"], "unit": head["unit"],
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": "u8",
               "data": "synthetic (seeded gradient+noise, synth/gen.py)",
               "config": head["config"], "roofline": head["roofline"],
               "per_transform": head["per_transform"], "trials": head["trials"], "cpu_baseline": cpu,
               "e2e": head["e2e"],
               "gpu_launches": head["gpu_launches"] + sum(c["gpu_launches"] for c in composed.values()),
               "clocks": head["clocks"]}
        if composed:
            out["composed"] = composed
        print(json.dumps(out))
    if dist:
        dist.destroy_process_group()


def run_reference(args, world, rank):
    """--impl reference: the oracle as it stands, on the host cores, bounded.
    Same config object, metric and unit as our arm's headline line (cfg2 by
    default), so the driver's ratios compare like with like; each step is a
    bounded sample of that workload (stated in cpu_baseline.sample)."""
    if rank != 0:
        return
    cfg = 2 if args.config == 0 else args.config
    name, menu, sizes, _ = workload(cfg, 0)
    threads = os.cpu_count() or 1
    n_img = 256 if cfg == 2 else 4
    for s in range(args.warmup):
        oracle_menu_rate(menu, sizes, 2, args.seed + s, threads)
    t = 0.0
    for s in range(args.steps):
        _, dt = oracle_menu_rate(menu, sizes, n_img, args.seed + s, threads)
        t += dt
    val = n_img * args.steps / t
    unit = unit_of(cfg, menu)
    out = {"impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": unit,
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(t / args.steps * 1e3, 2), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_dict(cfg, name, sizes, world),
           "cpu_baseline": {"value": round(val, 3), "unit": unit, "cores": threads,
                            "kind": "oracle",
                            "sample": "each step = first %d images of the workload through the "
                                      "whole menu, plain C oracle on %d host threads"
                                      % (n_img, threads)},
           "e2e": {"value": round(val, 3), "unit": unit, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
