// abi.cu -- the C ABI (include/alb_b200.h): pipeline validation, batch
// layouts, the launch planner (fusion into rowgather / resample / affine /
// pointwise / equalize steps) and the stream-ordered launch sequence.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "config.h"
#include "kernels.cuh"
#include "stages.cuh"

using namespace alb;

#ifndef ALB_Q4_BUDGET_KB
#define ALB_Q4_BUDGET_KB 72  // shared-memory budget of one quad-resample CTA (sets the band height)
#endif
#ifndef ALB_Q4_MAXRC
#define ALB_Q4_MAXRC 4  // largest quad-resample band height 4 << rc
#endif
#ifndef ALB_Q4_BANDS
#define ALB_Q4_BANDS 8  // bands of one quad-resample unit (a CTA prefetches band b + 1 while computing b)
#endif
static_assert(ALB_Q4_BANDS >= 1 && ALB_Q4_BANDS <= 16, "the quad-resample kernel keeps <= 16 bands' window rows");

namespace {

thread_local std::string g_err;

alb_status fail(alb_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_TRY(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) return fail(ALB_E_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)

bool is_shape_kind(int k) {
  return k == ALB_RANDOM_CROP || k == ALB_PAD_TO_SIZE || k == ALB_RESIZE ||
         k == ALB_RANDOM_SIZED_CROP || k == ALB_CROP;
}
bool is_exact_kind(int k) {
  return k == ALB_HFLIP || k == ALB_VFLIP || k == ALB_CROP || k == ALB_RANDOM_CROP ||
         k == ALB_PAD_TO_SIZE;
}
bool is_rgb_only(int k) {
  return k == ALB_SHIFT_RGB || k == ALB_SHIFT_HSV || k == ALB_GRAYSCALE || k == ALB_NORMALIZE;
}

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

struct alb_pipeline {
  std::vector<alb_op> ops;
};

struct alb_layout {
  std::vector<alb_image_desc> h;
  alb_image_desc* d = nullptr;
  int n = 0, channels = 3;
  size_t span = 0;  // bytes from offset 0 to the end of the last image
  ~alb_layout() {
    if (d) cudaFree(d);
  }
};

namespace {

enum StepKind { SK_ROW = 0, SK_POINT = 1, SK_RESAMPLE = 2, SK_AFFINE = 3, SK_EQ = 4, SK_D4 = 5, SK_ELASTIC = 6 };
enum BufId { B_IN = 0, B_OUT = 1, B_WS0 = 2, B_WS1 = 3, B_NONE = 4 };

struct PlanStep {
  StepKind kind;
  int slot0 = 0, slot1 = 0;
  std::vector<Stage> stages;
  bool normalize = false;
  bool has_image = true;   // ROW step may be mask-only
  bool has_mask = false;
  int src = B_IN, dst = B_OUT, msrc = B_NONE, mdst = B_NONE;
  const alb_layout* src_l = nullptr;
  const alb_layout* dst_l = nullptr;
  const alb_layout* msrc_l = nullptr;
  const alb_layout* mdst_l = nullptr;
  std::vector<int2> units, munits;
  size_t units_off = 0, munits_off = 0;  // into the plan's device unit table
  std::vector<int> ustart, mstart;       // first unit (mask unit) of image i, size n + 1
  int unit_size = 0, munit_size = 0, unit_rows = 0;
  bool flat = false;
  uint32_t fill = 0, mask_fill = 0;
  int interp = 1, border = 0;
  int eq_slot = -1;
  float min_scale = 1.0f;
  int rs_ring = 0, rs_sw = 0, rs_hw = 0;  // separable resample parameters (0 = old kernel)
  int rs_q = 0;                           // quad-column resample: staged rows per unit (0 = off)
  int self_sample = 0;                    // the kernel draws its images' params itself (no K0)
  int g_r = 0, g_off = 0;                  // ElasticTransform radius, weights offset in d_gauss
  double alpha = 0.0;
};

constexpr int kChunk = 48 * 512;         // pointwise / histogram bytes per unit
#ifndef ALB_LUT_CHUNK
#define ALB_LUT_CHUNK 245760
#endif
#ifndef ALB_PX_CHUNK
#define ALB_PX_CHUNK 122880
#endif
// pointwise step bytes per unit (multiples of 48): LUT-only steps restage the
// image's LUTs per unit, so their units are larger
constexpr int kLutChunk = ALB_LUT_CHUNK, kPxChunk = ALB_PX_CHUNK;
constexpr int kStageWords = 10 * 1024;   // resample staging capacity (40 KB)

}  // namespace

struct alb_plan {
  std::vector<alb_op> ops;
  alb_op* d_ops = nullptr;
  int n = 0;
  const alb_layout* in = nullptr;
  const alb_layout* out = nullptr;
  const alb_layout* min = nullptr;
  const alb_layout* mout = nullptr;
  std::vector<std::unique_ptr<alb_layout>> inter;  // intermediate layouts
  std::vector<PlanStep> steps;
  int n_luts = 0;
  int lut_k0[kMaxLuts], lut_k1[kMaxLuts];
  int norm_slot = -1;
  int out_h = 0, out_w = 0;  // NCHW dims
  int max_boxes = 0;
  float min_vis = 0.f;
  bool has_eq = false;
  // workspace layout
  size_t off_params = 0, off_fired = 0, off_dims = 0, off_luts = 0, off_norm = 0,
         off_eqh = 0, off_eql = 0, off_buf[2] = {0, 0}, off_mbuf[2] = {0, 0}, off_geo = 0, off_tiles = 0, off_grid = 0,
         ws_bytes = 0;
  int n_grid = 0;  // GridDistortion slots (per-image knot tables in the workspace)
  std::vector<double> gauss;  // ElasticTransform weights of every elastic step (host copy)
  double* d_gauss = nullptr;
  int2* d_units = nullptr;
  int n_launches = 0;
  // alb_apply_host pipeline: copy streams and per-chunk events (created on first use)
  mutable cudaStream_t s_in = nullptr, s_out = nullptr;
  mutable std::vector<cudaEvent_t> ev;
  ~alb_plan() {
    if (d_ops) cudaFree(d_ops);
    if (d_gauss) cudaFree(d_gauss);
    if (d_units) cudaFree(d_units);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
  }
};

// ------------------------------------------------------------------ helpers

static alb_status validate_ops(const alb_op* ops, int n_ops) {
  if (n_ops < 0 || (n_ops > 0 && !ops)) return fail(ALB_E_INVALID_ARG, "null op list");
  if (n_ops > ALB_MAX_OPS) return fail(ALB_E_UNSUPPORTED, "more than ALB_MAX_OPS ops");
  for (int k = 0; k < n_ops; ++k) {
    const alb_op& o = ops[k];
    const std::string at = "op " + std::to_string(k) + ": ";
    if (o.kind < 0 || o.kind >= ALB_NUM_KINDS) return fail(ALB_E_UNKNOWN_OP, at + "unknown kind");
    if (!(o.p >= 0.0 && o.p <= 1.0)) return fail(ALB_E_RANGE, at + "p outside [0,1]");
    for (int j = 0; j < 4; ++j)
      if (!(o.lo[j] <= o.hi[j])) return fail(ALB_E_RANGE, at + "lo > hi");
    if (is_shape_kind(o.kind) && o.p != 1.0)
      return fail(ALB_E_RANGE, at + "shape-changing ops require p == 1 (R17)");
    if (o.interp != ALB_INTERP_NEAREST && o.interp != ALB_INTERP_BILINEAR)
      return fail(ALB_E_RANGE, at + "bad interp");
    if (o.border != ALB_BORDER_CONSTANT && o.border != ALB_BORDER_REFLECT_101)
      return fail(ALB_E_RANGE, at + "bad border");
    switch (o.kind) {
      case ALB_SHIFT_SCALE_ROTATE:
        if (!(o.lo[2] > 0.0)) return fail(ALB_E_RANGE, at + "scale <= 0");
        break;
      case ALB_BRIGHTNESS: case ALB_CONTRAST:
        if (!(o.lo[0] >= 0.0)) return fail(ALB_E_RANGE, at + "negative factor");
        break;
      case ALB_BRIGHTNESS_CONTRAST:
        if (!(o.lo[0] >= 0.0) || !(o.lo[1] >= 0.0)) return fail(ALB_E_RANGE, at + "negative factor");
        break;
      case ALB_GAMMA:
        if (!(o.lo[0] > 0.0)) return fail(ALB_E_RANGE, at + "gamma <= 0");
        break;
      case ALB_RANDOM_CROP: case ALB_CROP: case ALB_PAD_TO_SIZE: case ALB_RESIZE:
        if (o.out_w < 1 || o.out_h < 1) return fail(ALB_E_RANGE, at + "output size < 1");
        break;
      case ALB_RANDOM_SIZED_CROP:
        if (o.out_w < 1 || o.out_h < 1 || o.min_side < 1 || o.max_side < o.min_side)
          return fail(ALB_E_RANGE, at + "bad RandomSizedCrop sides");
        break;
      case ALB_ROT90: case ALB_D4: {
        const double top = o.kind == ALB_ROT90 ? 3.0 : 7.0;
        if (!(o.lo[0] >= 0.0 && o.hi[0] <= top) || std::floor(o.lo[0]) != o.lo[0] ||
            std::floor(o.hi[0]) != o.hi[0])
          return fail(ALB_E_RANGE, at + "element range must be integers within the group");
        break;
      }
      case ALB_ELASTIC:  // fixed alpha >= 0, sigma in (0, 16] (reading R32)
        if (o.lo[0] != o.hi[0] || o.lo[1] != o.hi[1]) return fail(ALB_E_RANGE, at + "alpha / sigma must be fixed");
        if (!(o.lo[0] >= 0.0)) return fail(ALB_E_RANGE, at + "alpha < 0");
        if (!(o.lo[1] > 0.0 && o.lo[1] <= 16.0)) return fail(ALB_E_RANGE, at + "sigma outside (0, 16]");
        break;
      case ALB_GRID_DISTORTION:  // every step factor 1 + U(lo, hi) stays > 0
        if (o.num_steps < 1 || o.num_steps > ALB_GRID_MAX_STEPS)
          return fail(ALB_E_RANGE, at + "num_steps outside [1, 32]");
        if (!(o.lo[0] > -1.0 && o.hi[0] < 1.0)) return fail(ALB_E_RANGE, at + "distort limit outside (-1, 1)");
        break;
      case ALB_NORMALIZE:
        if (k != n_ops - 1 || o.p != 1.0) return fail(ALB_E_RANGE, at + "Normalize must be last, p = 1");
        for (int c = 0; c < 3; ++c)
          if (!(o.std[c] != 0.0)) return fail(ALB_E_RANGE, at + "std == 0");
        break;
      default: break;
    }
  }
  return ALB_OK;
}

// GridDistortion: largest source/destination slope of an axis map, n f_i / S
// <= (1 + hi) / (1 + lo) (reading R31), with a margin for rounding
static double grid_stretch(const alb_op& o) { return (1.0 + o.hi[0]) / (1.0 + o.lo[0]) * (1.0 + 1e-9); }

// dims each slot sees for an h x w input; error if a window does not fit
static alb_status track_dims(const std::vector<alb_op>& ops, int h, int w,
                             std::vector<std::pair<int, int>>& dims) {
  dims.clear();
  for (size_t k = 0; k < ops.size(); ++k) {
    dims.push_back({h, w});
    const alb_op& o = ops[k];
    switch (o.kind) {
      case ALB_RANDOM_CROP:
        if (o.out_w > w || o.out_h > h) return fail(ALB_E_INVALID_ARG, "RandomCrop larger than image");
        h = o.out_h; w = o.out_w; break;
      case ALB_CROP:
        if (o.crop_x < 0 || o.crop_y < 0 || o.crop_x + o.out_w > w || o.crop_y + o.out_h > h)
          return fail(ALB_E_INVALID_ARG, "Crop window outside the image");
        h = o.out_h; w = o.out_w; break;
      case ALB_PAD_TO_SIZE:
        if (w > o.out_w || h > o.out_h) return fail(ALB_E_INVALID_ARG, "PadToSize target smaller than image");
        h = o.out_h; w = o.out_w; break;
      case ALB_RESIZE:
        h = o.out_h; w = o.out_w; break;
      case ALB_RANDOM_SIZED_CROP:
        if (o.min_side > std::min(h, w)) return fail(ALB_E_INVALID_ARG, "RandomSizedCrop min side > image");
        h = o.out_h; w = o.out_w; break;
      case ALB_ROT90: case ALB_D4: {
        // the shape must not depend on the draw (reading R30)
        bool can_odd = false, can_even = o.p < 1.0;
        for (int e = (int)o.lo[0]; e <= (int)o.hi[0]; ++e) (e & 1 ? can_odd : can_even) = true;
        if (can_odd && can_even && h != w)
          return fail(ALB_E_UNSUPPORTED, "Rot90/D4 whose parity varies on a non-square image");
        if (can_odd) std::swap(h, w);
        break;
      }
      default: break;
    }
  }
  dims.push_back({h, w});
  return ALB_OK;
}

static alb_status upload_layout(alb_layout* l) {
  l->span = 0;
  for (auto& d : l->h) l->span = std::max(l->span, (size_t)(d.offset + (int64_t)d.height * d.pitch));
  if (l->d) { cudaFree(l->d); l->d = nullptr; }
  if (l->n > 0) {
    CUDA_TRY(cudaMalloc(&l->d, sizeof(alb_image_desc) * l->n));
    CUDA_TRY(cudaMemcpy(l->d, l->h.data(), sizeof(alb_image_desc) * l->n, cudaMemcpyHostToDevice));
  }
  return ALB_OK;
}

// packed 256-aligned layout for intermediate images
static alb_status make_packed(const std::vector<std::pair<int, int>>& hw, int channels,
                              std::unique_ptr<alb_layout>& out) {
  out.reset(new alb_layout);
  out->n = (int)hw.size();
  out->channels = channels;
  int64_t off = 0;
  for (auto& p : hw) {
    alb_image_desc d{};
    d.offset = off;
    d.height = p.first;
    d.width = p.second;
    d.pitch = p.second * channels;
    out->h.push_back(d);
    off = (int64_t)align_up((size_t)(off + (int64_t)d.height * d.pitch), 256);
  }
  return upload_layout(out.get());
}

static void row_units(PlanStep& st, const alb_layout* dst, int channels, std::vector<int2>& u,
                      int& usize) {
  int wmax = 1;
  for (auto& d : dst->h) wmax = std::max(wmax, d.width);
  const int nbmax = 2 + wmax / 16;
  usize = std::max(1, 2048 / nbmax);  // ~8 blocks of 16 px per thread (measured: 2048 > 1024, 4096)
  (void)channels;
  (void)st;
  for (int i = 0; i < dst->n; ++i)
    for (int y = 0; y < dst->h[i].height; y += usize) u.push_back(make_int2(i, y / usize));
}

// ----------------------------------------------------------------- the ABI

// Launch the plan's kernels for images [i0, i1) (alb_apply: the whole batch;
// alb_apply_host: chunks, so copies and kernels of different chunks overlap).
// Every kernel either iterates per-image (K0, affine setup, equalize LUT) over
// the range or takes the range's contiguous slice of its step's unit table.
static alb_status launch_range(const alb_plan* P, uint64_t seed, uint64_t first_image_index,
                               const uint8_t* img_in, uint8_t* img_out, float* out_nchw,
                               const uint8_t* mask_in, uint8_t* mask_out, const float* boxes_in,
                               const int32_t* labels_in, const int32_t* count_in, float* boxes_out,
                               int32_t* labels_out, int32_t* count_out, uint8_t* ws, int i0, int i1,
                               cudaStream_t stream) {
  const int n_ops = (int)P->ops.size();

  Tables tab{};
  tab.params = (const double*)(ws + P->off_params);
  tab.fired = ws + P->off_fired;
  tab.dims = (const int32_t*)(ws + P->off_dims);
  tab.luts = ws + P->off_luts;
  tab.norm_lut = (const float*)(ws + P->off_norm);
  tab.eq_luts = ws + P->off_eql;
  tab.n_ops = n_ops;
  tab.n_luts = P->n_luts;
  tab.grid = (const double*)(ws + P->off_grid);
  tab.n_grid = P->n_grid;

  PrepArgs pa{};
  pa.ops = P->d_ops;
  pa.n_ops = n_ops;
  pa.n = i1 - i0;
  pa.img0 = i0;
  pa.seed = seed;
  pa.first_image = (uint32_t)first_image_index;
  pa.in_desc = P->in->d;
  pa.params = (double*)(ws + P->off_params);
  pa.fired = ws + P->off_fired;
  pa.dims = (int32_t*)(ws + P->off_dims);
  pa.luts = ws + P->off_luts;
  pa.n_luts = P->n_luts;
  for (int s = 0; s < P->n_luts; ++s) { pa.lut_k0[s] = P->lut_k0[s]; pa.lut_k1[s] = P->lut_k1[s]; }
  pa.norm_lut = (float*)(ws + P->off_norm);
  pa.norm_slot = P->norm_slot;
  pa.grid = (double*)(ws + P->off_grid);
  pa.n_grid = P->n_grid;
  // K0, unless the plan's only step is an integer geometric map whose kernel
  // draws its images' params itself (flips / crops / pads: one launch)
  if (!(P->steps.size() == 1 && P->steps[0].self_sample)) launch_prep(pa, stream);
  if (P->max_boxes > 0) {  // (boxes only on full-range launches; side stream, beside the pixel steps)
    BoxArgs b{};
    b.boxes_in = boxes_in;
    b.labels_in = labels_in;
    b.count_in = count_in;
    b.boxes_out = boxes_out;
    b.labels_out = labels_out;
    b.count_out = count_out;
    b.max_boxes = P->max_boxes;
    b.min_visibility = P->min_vis;
    b.n = P->n;
    b.tab = tab;
    b.ops = P->d_ops;
    launch_boxes(b, side_fork(stream));
  }

  auto img_buf = [&](int id) -> uint8_t* {
    switch (id) {
      case B_IN: return const_cast<uint8_t*>(img_in);
      case B_OUT: return img_out;
      case B_WS0: return ws + P->off_buf[0];
      case B_WS1: return ws + P->off_buf[1];
      default: return nullptr;
    }
  };
  auto mask_buf = [&](int id) -> uint8_t* {
    switch (id) {
      case B_IN: return const_cast<uint8_t*>(mask_in);
      case B_OUT: return mask_out;
      case B_WS0: return ws + P->off_mbuf[0];
      case B_WS1: return ws + P->off_mbuf[1];
      default: return nullptr;
    }
  };

  for (size_t si = 0; si < P->steps.size(); ++si) {
    const PlanStep& st = P->steps[si];
    StepArgs a{};
    a.src = img_buf(st.src);
    a.sdesc = st.src_l ? st.src_l->d : nullptr;
    a.dst = img_buf(st.dst);
    a.ddesc = st.dst_l ? st.dst_l->d : nullptr;
    a.nchw = st.normalize ? out_nchw : nullptr;
    a.out_h = P->out_h;
    a.out_w = P->out_w;
    a.msrc = st.has_mask ? mask_buf(st.msrc) : nullptr;
    a.msdesc = st.has_mask ? st.msrc_l->d : nullptr;
    a.mdst = st.has_mask ? mask_buf(st.mdst) : nullptr;
    a.mddesc = st.has_mask ? st.mdst_l->d : nullptr;
    a.units = P->d_units + st.units_off + st.ustart[i0];
    a.n_units = st.ustart[i1] - st.ustart[i0];
    a.unit_size = st.unit_size;
    a.unit_rows = st.unit_rows;
    a.slot0 = st.slot0;
    a.slot1 = st.slot1;
    a.n_stages = (int)st.stages.size();
    for (int s = 0; s < a.n_stages; ++s) a.stages[s] = st.stages[s];
    a.normalize = st.normalize ? 1 : 0;
    a.flat = st.flat ? 1 : 0;
    a.fill = st.fill;
    a.mask_fill = st.mask_fill;
    a.interp = st.interp;
    a.border = st.border;
    a.min_scale = st.min_scale;
    a.tab = tab;
    a.ops = P->d_ops;
    a.geo = ws + P->off_geo;
    a.tiles = st.kind == SK_AFFINE ? ws + P->off_tiles + (st.units_off + st.ustart[i0]) * kAffSub * kTileInfoBytes : nullptr;
    a.img0 = i0;
    a.n_img = i1;
    a.rs_ring = st.rs_ring;
    a.rs_sw = st.rs_sw;
    a.rs_hw = st.rs_hw;
    a.rs_q = st.rs_q;
    a.self_sample = st.self_sample;
    a.lut_k0 = a.lut_k1 = 0;
    if (st.self_sample && st.kind == SK_POINT && st.stages[0].type == ST_LUT) {
      a.lut_k0 = P->lut_k0[st.stages[0].lut];
      a.lut_k1 = P->lut_k1[st.stages[0].lut];
    }
    a.seed = seed;
    a.first_image = (uint32_t)first_image_index;
    a.gauss = P->d_gauss ? P->d_gauss + st.g_off : nullptr;
    a.g_r = st.g_r;
    a.alpha = st.alpha;
    cudaStream_t ms;
    switch (st.kind) {
      case SK_ROW:
        a.rg_wide = st.slot1 > st.slot0 ? 2 : 0;
        for (int k = st.slot0; k < st.slot1; ++k) {
          const int kd = P->ops[k].kind;
          if (kd == ALB_PAD_TO_SIZE || kd == ALB_CROP || kd == ALB_RANDOM_CROP) a.rg_wide = 1;
          else if (kd != ALB_HFLIP && kd != ALB_VFLIP && a.rg_wide == 2) a.rg_wide = 0;
        }
        // labels on the side stream (forked before the pixels launch), beside the pixels
        ms = st.has_mask && st.has_image ? side_fork(stream) : stream;
        if (st.has_image) {
          a.channels = 3;
          launch_rowgather(a, stream);
        }
        if (st.has_mask) {
          a.channels = 1;
          a.units = P->d_units + st.munits_off + st.mstart[i0];
          a.n_units = st.mstart[i1] - st.mstart[i0];
          a.unit_size = st.munit_size;
          launch_rowgather(a, ms);
          if (ms != stream) side_join(stream);
        }
        break;
      case SK_POINT: {
        // 16-byte co-alignment of source and destination segments
        bool vec = true;
        if (a.dst) {
          for (int i = 0; i < P->n && vec; ++i) {
            const uintptr_t s = (uintptr_t)a.src + st.src_l->h[i].offset;
            const uintptr_t d = (uintptr_t)a.dst + st.dst_l->h[i].offset;
            vec = ((s ^ d) & 15) == 0 && (st.flat || ((st.src_l->h[i].pitch - st.dst_l->h[i].pitch) % 16) == 0);
          }
        }
        a.vec_ok = vec ? 1 : 0;
        launch_point(a, stream);
        break;
      }
      case SK_RESAMPLE: launch_resample(a, stream); break;
      case SK_AFFINE: launch_affine(a, stream); break;
      case SK_ELASTIC: launch_elastic(a, stream); break;
      case SK_D4:
        ms = st.has_mask && st.has_image ? side_fork(stream) : stream;
        if (st.has_image) {
          a.channels = 3;
          launch_d4(a, stream);
        }
        if (st.has_mask) {
          a.channels = 1;
          a.units = P->d_units + st.munits_off + st.mstart[i0];
          a.n_units = st.mstart[i1] - st.mstart[i0];
          launch_d4(a, ms);
          if (ms != stream) side_join(stream);
        }
        break;
      case SK_EQ: {
        // single-pass Equalize when its LUT pass is a plain packed, co-aligned
        // pointwise step holding only the Equalize stage (K8, one kernel)
        if (si + 1 < P->steps.size()) {
          const PlanStep& ap = P->steps[si + 1];
          bool fuse = ap.kind == SK_POINT && ap.stages.size() == 1 && ap.stages[0].type == ST_EQ &&
                      !ap.normalize && ap.flat && ap.src == st.src;
          uint8_t* dst = img_buf(ap.dst);
          for (int i = i0; i < i1 && fuse; ++i) {
            const uintptr_t sp = (uintptr_t)a.src + st.src_l->h[i].offset;
            const uintptr_t dp = (uintptr_t)dst + ap.dst_l->h[i].offset;
            fuse = ((sp ^ dp) & 15) == 0;
          }
          if (fuse) {
            StepArgs f = a;
            f.dst = dst;
            f.ddesc = ap.dst_l->d;
            f.n_stages = 1;
            f.stages[0] = ap.stages[0];
            f.flat = 1;
            f.vec_ok = 1;
            f.normalize = 0;
            launch_eq_fused(f, stream);
            ++si;  // the LUT pass ran inside
            break;
          }
        }
        EqArgs e{};
        e.src = a.src;
        e.sdesc = a.sdesc;
        e.hist = (uint32_t*)(ws + P->off_eqh);
        e.lut = ws + P->off_eql;
        e.units = a.units;
        e.n_units = a.n_units;
        e.unit_size = st.flat ? -1 : 0;  // -1: whole flat images (k_eq_hist_lane)
        e.n = i1 - i0;
        e.img0 = i0;
        e.slot = st.eq_slot;
        e.tab = tab;
        // a failed memset must still join the box work forked above before
        // returning (else the caller's stream is not ordered after it)
        const cudaError_t me = cudaMemsetAsync(e.hist + (size_t)i0 * 768, 0,
                                               (size_t)(i1 - i0) * 768 * sizeof(uint32_t), stream);
        if (me != cudaSuccess) {
          if (P->max_boxes > 0) side_join(stream);
          return fail(ALB_E_CUDA, std::string("memset failed: ") + cudaGetErrorString(me));
        }
        launch_eq_hist(e, stream);
        launch_eq_lut(e, stream);
        break;
      }
    }
  }
  if (P->max_boxes > 0) side_join(stream);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ALB_E_CUDA, std::string("launch failed: ") + cudaGetErrorString(e));
  return ALB_OK;
}

namespace alb {
alb_status set_error(alb_status s, const std::string& msg) { return fail(s, msg); }
const std::vector<alb_op>& pipeline_ops(const alb_pipeline* p) { return p->ops; }
const std::vector<alb_image_desc>& layout_desc(const alb_layout* l) { return l->h; }
int layout_channels(const alb_layout* l) { return l->channels; }
}  // namespace alb

extern "C" {

const char* alb_last_error(void) { return g_err.c_str(); }
int32_t alb_version(void) { return 1; }

alb_status alb_pipeline_create(const alb_op* ops, int32_t n_ops, alb_pipeline** out) {
  if (!out) return fail(ALB_E_INVALID_ARG, "null out");
  alb_status s = validate_ops(ops, n_ops);
  if (s) return s;
  auto* p = new alb_pipeline;
  p->ops.assign(ops, ops + n_ops);
  *out = p;
  return ALB_OK;
}

void alb_pipeline_destroy(alb_pipeline* p) { delete p; }

alb_status alb_output_shape(const alb_pipeline* p, int32_t in_h, int32_t in_w, int32_t* out_h,
                            int32_t* out_w) {
  if (!p || !out_h || !out_w) return fail(ALB_E_INVALID_ARG, "null argument");
  if (in_h < 1 || in_w < 1) return fail(ALB_E_SHAPE, "image dims < 1");
  std::vector<std::pair<int, int>> dims;
  alb_status s = track_dims(p->ops, in_h, in_w, dims);
  if (s) return s;
  *out_h = dims.back().first;
  *out_w = dims.back().second;
  return ALB_OK;
}

alb_status alb_layout_create(const alb_image_desc* desc, int32_t n, int32_t channels,
                             alb_layout** out) {
  if (!out || n < 0 || (n > 0 && !desc)) return fail(ALB_E_INVALID_ARG, "bad layout arguments");
  if (channels != 1 && channels != 3) return fail(ALB_E_UNSUPPORTED, "channels must be 1 or 3");
  for (int i = 0; i < n; ++i) {
    if (desc[i].height < 1 || desc[i].width < 1) return fail(ALB_E_SHAPE, "image dims < 1");
    if (desc[i].offset < 0 || desc[i].pitch < desc[i].width * channels)
      return fail(ALB_E_ALIGN, "negative offset or pitch < width*channels");
  }
  std::unique_ptr<alb_layout> l(new alb_layout);
  l->h.assign(desc, desc + n);
  l->n = n;
  l->channels = channels;
  alb_status s = upload_layout(l.get());
  if (s) return s;
  *out = l.release();
  return ALB_OK;
}

void alb_layout_destroy(alb_layout* l) { delete l; }

alb_status alb_plan_create(const alb_pipeline* p, const alb_layout* in, const alb_layout* out,
                           const alb_layout* mask_in, const alb_layout* mask_out,
                           int32_t max_boxes, float min_visibility, alb_plan** plan_out) {
  if (!p || !in || !plan_out) return fail(ALB_E_INVALID_ARG, "null argument");
  if (in->channels != 3) return fail(ALB_E_UNSUPPORTED, "images must have 3 channels");
  if ((mask_in == nullptr) != (mask_out == nullptr)) return fail(ALB_E_INVALID_ARG, "mask_in/mask_out must both be set");
  if (max_boxes < 0) return fail(ALB_E_INVALID_ARG, "max_boxes < 0");
  for (const alb_op& o : p->ops)
    if ((o.kind == ALB_GRID_DISTORTION || o.kind == ALB_ELASTIC) && max_boxes > 0)
      return fail(ALB_E_UNSUPPORTED, "boxes under a free-form warp (GridDistortion / ElasticTransform)");
  std::unique_ptr<alb_plan> P(new alb_plan);
  P->ops = p->ops;
  P->n = in->n;
  P->in = in; P->out = out; P->min = mask_in; P->mout = mask_out;
  P->max_boxes = max_boxes;
  P->min_vis = min_visibility;
  const int n_ops = (int)P->ops.size();
  const bool ends_norm = n_ops > 0 && P->ops.back().kind == ALB_NORMALIZE;
  if (ends_norm != (out == nullptr)) return fail(ALB_E_INVALID_ARG, "out must be NULL iff the pipeline ends in Normalize");
  if (out && out->n != in->n) return fail(ALB_E_SHAPE, "in/out batch sizes differ");
  if (out && out->channels != 3) return fail(ALB_E_SHAPE, "out must have 3 channels");
  if (mask_in && (mask_in->n != in->n || mask_out->n != in->n || mask_in->channels != 1 || mask_out->channels != 1))
    return fail(ALB_E_SHAPE, "mask layouts must be 1-channel with the same count");

  // per-image dims through the pipeline
  std::vector<std::vector<std::pair<int, int>>> dims(P->n);
  for (int i = 0; i < P->n; ++i) {
    alb_status s = track_dims(P->ops, in->h[i].height, in->h[i].width, dims[i]);
    if (s) return s;
    const auto& f = dims[i].back();
    if (out && (out->h[i].height != f.first || out->h[i].width != f.second))
      return fail(ALB_E_SHAPE, "output layout dims differ from the pipeline's output shape (image " + std::to_string(i) + ")");
    if (ends_norm) {
      if (i == 0) { P->out_h = f.first; P->out_w = f.second; }
      else if (P->out_h != f.first || P->out_w != f.second)
        return fail(ALB_E_SHAPE, "Normalize output needs one output size for the batch");
    }
    if (mask_in) {
      if (mask_in->h[i].height != in->h[i].height || mask_in->h[i].width != in->h[i].width)
        return fail(ALB_E_SHAPE, "mask dims differ from image dims (SPEC.md:47)");
      if (mask_out->h[i].height != f.first || mask_out->h[i].width != f.second)
        return fail(ALB_E_SHAPE, "mask output dims differ from the output shape");
    }
  }
  // identity resizes (input dims == output dims for every image) are no-ops
  std::vector<bool> ident(n_ops, false);
  for (int k = 0; k < n_ops; ++k) {
    if (P->ops[k].kind != ALB_RESIZE) continue;
    bool all = true;
    for (int i = 0; i < P->n && all; ++i) all = dims[i][k] == dims[i][k + 1];
    ident[k] = all;
  }

  // ---------------------------------------------------------- group ops
  std::vector<PlanStep>& steps = P->steps;
  int k = 0;
  bool geo_open = false;  // last step is resample/affine still accepting post exact ops
  bool point_open = false;
  while (k < n_ops) {
    const alb_op& o = P->ops[k];
    const int kind = o.kind;
    if (kind == ALB_NORMALIZE) {
      if (!steps.empty() && (steps.back().kind == SK_POINT || steps.back().kind == SK_RESAMPLE ||
                             steps.back().kind == SK_AFFINE) && (point_open || geo_open)) {
        steps.back().normalize = true;
      } else {
        PlanStep st; st.kind = SK_POINT; st.slot0 = k; st.slot1 = k; st.normalize = true;
        steps.push_back(st);
      }
      P->norm_slot = k;
      ++k;
      geo_open = point_open = false;
      continue;
    }
    if (is_exact_kind(kind) || (kind == ALB_RESIZE && ident[k])) {
      if (geo_open && kind != ALB_PAD_TO_SIZE) {  // fuse as a post op (commutes with stages)
        steps.back().slot1 = k + 1;
        ++k;
        continue;
      }
      PlanStep st; st.kind = SK_ROW; st.slot0 = k;
      int pads = 0;
      int j = k;
      while (j < n_ops && (is_exact_kind(P->ops[j].kind) || (P->ops[j].kind == ALB_RESIZE && ident[j]))) {
        if (P->ops[j].kind == ALB_PAD_TO_SIZE) {
          if (pads == 1) break;
          ++pads;
          st.fill = P->ops[j].fill[0] | (P->ops[j].fill[1] << 8) | (P->ops[j].fill[2] << 16);
          st.mask_fill = P->ops[j].mask_fill;
        }
        ++j;
      }
      st.slot1 = j;
      steps.push_back(st);
      k = j;
      geo_open = point_open = false;
      continue;
    }
    if (kind == ALB_ELASTIC) {  // field + remap, own step (post ops start a new step)
      PlanStep st; st.kind = SK_ELASTIC; st.slot0 = k; st.slot1 = k + 1;
      st.interp = o.interp; st.border = o.border;
      st.fill = o.fill[0] | (o.fill[1] << 8) | (o.fill[2] << 16);
      st.mask_fill = o.mask_fill;
      // normalised truncated Gaussian, ascending-k sum (reading R32)
      const double sigma = o.lo[1];
      const int r = (int)std::ceil(3.0 * sigma);
      st.g_r = r;
      st.g_off = (int)P->gauss.size();
      st.alpha = o.lo[0];
      std::vector<double> g(2 * r + 1);
      double sum = 0.0;
      for (int q = -r; q <= r; ++q) {
        g[q + r] = std::exp(-(double)(q * q) / (2.0 * sigma * sigma));
        sum += g[q + r];
      }
      for (double& v : g) P->gauss.push_back(v / sum);
      steps.push_back(st);
      ++k;
      geo_open = point_open = false;
      continue;
    }
    if (kind == ALB_ROT90 || kind == ALB_D4) {  // signed permutation, own step
      PlanStep st; st.kind = SK_D4; st.slot0 = k; st.slot1 = k + 1;
      steps.push_back(st);
      ++k;
      geo_open = point_open = false;
      continue;
    }
    if (kind == ALB_RESIZE || kind == ALB_RANDOM_SIZED_CROP || kind == ALB_ROTATE ||
        kind == ALB_SHIFT_SCALE_ROTATE || kind == ALB_GRID_DISTORTION) {
      PlanStep st;
      st.kind = (kind == ALB_ROTATE || kind == ALB_SHIFT_SCALE_ROTATE) ? SK_AFFINE : SK_RESAMPLE;
      st.slot0 = k; st.slot1 = k + 1;
      st.interp = o.interp; st.border = o.border;
      st.min_scale = kind == ALB_SHIFT_SCALE_ROTATE ? (float)o.lo[2] : 1.0f;
      st.fill = o.fill[0] | (o.fill[1] << 8) | (o.fill[2] << 16);
      st.mask_fill = o.mask_fill;
      steps.push_back(st);
      ++k;
      geo_open = true;
      point_open = false;
      continue;
    }
    if (is_lut_kind(kind) || kind == ALB_SHIFT_HSV || kind == ALB_GRAYSCALE) {
      // a step whose kernel already carries kMaxStages stages (or 4 LUT-type
      // stages: the shared-memory LUT budget) is closed; a new pointwise step
      // takes the rest of the chain
      bool full = false;
      if (geo_open || point_open) {
        int nl = 0;
        for (auto& sg : steps.back().stages) nl += (sg.type == ST_LUT || sg.type == ST_EQ);
        full = steps.back().stages.size() >= (size_t)kMaxStages || (is_lut_kind(kind) && nl >= 4);
      }
      if (!(geo_open || point_open) || full) {
        PlanStep st; st.kind = SK_POINT; st.slot0 = k; st.slot1 = k;
        steps.push_back(st);
        point_open = true;
        geo_open = false;
      }
      PlanStep& b = steps.back();
      if (b.stages.size() >= (size_t)kMaxStages) return fail(ALB_E_UNSUPPORTED, "too many pointwise stages");
      Stage sg{};
      sg.slot = k;
      if (is_lut_kind(kind)) {
        int j = k;
        while (j < n_ops && is_lut_kind(P->ops[j].kind)) ++j;
        if (P->n_luts >= kMaxLuts) return fail(ALB_E_UNSUPPORTED, "too many LUT stages");
        sg.type = ST_LUT;
        sg.lut = P->n_luts;
        P->lut_k0[P->n_luts] = k;
        P->lut_k1[P->n_luts] = j;
        P->n_luts++;
        b.stages.push_back(sg);
        k = j;
      } else {
        sg.type = kind == ALB_SHIFT_HSV ? ST_HSV : ST_GRAY;
        b.stages.push_back(sg);
        ++k;
      }
      continue;
    }
    if (kind == ALB_EQUALIZE) {
      // several Equalize ops run in stream order and reuse one histogram / LUT
      // workspace region (each SK_EQ step rebuilds it from its own input)
      PlanStep st; st.kind = SK_EQ; st.slot0 = k; st.slot1 = k + 1; st.eq_slot = k;
      steps.push_back(st);
      PlanStep ap; ap.kind = SK_POINT; ap.slot0 = k; ap.slot1 = k + 1;
      Stage sg{}; sg.type = ST_EQ; sg.slot = k;
      ap.stages.push_back(sg);
      steps.push_back(ap);
      P->has_eq = true;
      point_open = true;
      geo_open = false;
      ++k;
      continue;
    }
    return fail(ALB_E_UNKNOWN_OP, "unhandled op kind");
  }
  // a lone integer-map step (flips, crops, pads) samples its own params: no
  // LUT, Normalize table, grid knots or box tables are needed from K0
#ifndef ALB_NO_SELF_SAMPLE
  if (steps.size() == 1 && steps[0].kind == SK_ROW && P->n_luts == 0 && P->norm_slot < 0 && max_boxes == 0)
    steps[0].self_sample = 1;
  // ... and so does a lone one-LUT pointwise step (its CTAs build the LUT)
  if (steps.size() == 1 && steps[0].kind == SK_POINT && !steps[0].normalize && P->norm_slot < 0 &&
      max_boxes == 0 && P->n_luts == 1 && steps[0].stages.size() == 1 && steps[0].stages[0].type == ST_LUT)
    steps[0].self_sample = 1;
  // ... and a lone HSV / gray pointwise step (parameters only, no tables)
  if (steps.size() == 1 && steps[0].kind == SK_POINT && !steps[0].normalize && P->norm_slot < 0 &&
      max_boxes == 0 && P->n_luts == 0 && !steps[0].stages.empty() &&
      std::all_of(steps[0].stages.begin(), steps[0].stages.end(),
                  [](const Stage& g) { return g.type == ST_HSV || g.type == ST_GRAY; }))
    steps[0].self_sample = 1;
#endif
  // LUT count per step must fit shared memory (<= 4 stages of 24 KB)
  for (auto& st : steps) {
    int nl = 0;
    for (auto& sg : st.stages) nl += (sg.type == ST_LUT || sg.type == ST_EQ);
    if (nl > 4) return fail(ALB_E_UNSUPPORTED, "more than 4 LUT stages in one fused step");
  }
  // rgb-only ops need 3 channels: images are always 3-channel here.
  const bool has_geo = std::any_of(steps.begin(), steps.end(), [](const PlanStep& s) {
    return s.kind == SK_ROW || s.kind == SK_RESAMPLE || s.kind == SK_AFFINE || s.kind == SK_D4 ||
           s.kind == SK_ELASTIC;
  });
  // masks ride on geometric steps; without one, an identity mask copy
  if (mask_in && !has_geo) {
    PlanStep st; st.kind = SK_ROW; st.slot0 = 0; st.slot1 = 0; st.has_image = false;
    steps.push_back(st);
  }
  if (steps.empty()) {  // empty / all-identity pipeline: copy
    PlanStep st; st.kind = SK_ROW; st.slot0 = 0; st.slot1 = 0;
    steps.push_back(st);
  }
  // ----------------------------------------------------- buffers + layouts
  // output dims of each step per image
  const int ns = (int)steps.size();
  int last_img = -1, last_mask = -1;
  for (int s = 0; s < ns; ++s) {
    if (steps[s].has_image && steps[s].kind != SK_EQ) last_img = s;
    if (mask_in && steps[s].kind != SK_POINT && steps[s].kind != SK_EQ) last_mask = s;
  }
  int cur = B_IN, mcur = mask_in ? B_IN : B_NONE;
  const alb_layout* cur_l = in;
  const alb_layout* mcur_l = mask_in;
  int ping = 0, mping = 0;
  size_t max_inter = 0, max_minter = 0;
  for (int s = 0; s < ns; ++s) {
    PlanStep& st = steps[s];
    // image
    if (st.kind == SK_EQ) {
      st.src = cur; st.src_l = cur_l; st.dst = B_NONE;
    } else if (st.has_image) {
      st.src = cur; st.src_l = cur_l;
      if (s == last_img) {
        st.dst = ends_norm ? B_NONE : B_OUT;
        st.dst_l = out;
      } else {
        std::vector<std::pair<int, int>> hw(P->n);
        const int kk = st.kind == SK_POINT ? st.slot0 : st.slot1;
        for (int i = 0; i < P->n; ++i) hw[i] = st.kind == SK_POINT ? std::make_pair(cur_l->h[i].height, cur_l->h[i].width) : dims[i][kk];
        std::unique_ptr<alb_layout> L;
        alb_status e = make_packed(hw, 3, L);
        if (e) return e;
        max_inter = std::max(max_inter, L->span);
        st.dst = B_WS0 + ping; ping ^= 1;
        st.dst_l = L.get();
        P->inter.push_back(std::move(L));
      }
      cur = st.dst; cur_l = st.dst_l;
    }
    // mask
    if (mask_in && st.kind != SK_POINT && st.kind != SK_EQ) {
      st.has_mask = true;
      st.msrc = mcur; st.msrc_l = mcur_l;
      if (s == last_mask) {
        st.mdst = B_OUT; st.mdst_l = mask_out;
      } else {
        std::vector<std::pair<int, int>> hw(P->n);
        for (int i = 0; i < P->n; ++i) hw[i] = st.has_image ? dims[i][st.slot1] : dims[i][0];
        std::unique_ptr<alb_layout> L;
        alb_status e = make_packed(hw, 1, L);
        if (e) return e;
        max_minter = std::max(max_minter, L->span);
        st.mdst = B_WS0 + mping; mping ^= 1;
        st.mdst_l = L.get();
        P->inter.push_back(std::move(L));
      }
      mcur = st.mdst; mcur_l = st.mdst_l;
    }
  }
  // ----------------------------------------------------------- work units
  size_t total_units = 0;
  for (auto& st : steps) {
    switch (st.kind) {
      case SK_ROW:
        if (st.has_image) row_units(st, st.dst_l, 3, st.units, st.unit_size);
        if (st.has_mask) row_units(st, st.mdst_l, 1, st.munits, st.munit_size);
        break;
      case SK_POINT:
      case SK_EQ: {
        const alb_layout* sl = st.src_l;
        bool flat = true;
        for (int i = 0; i < P->n; ++i) {
          flat = flat && sl->h[i].pitch == sl->h[i].width * 3 && sl->h[i].offset % 16 == 0;
          if (st.kind == SK_POINT && st.dst_l)
            flat = flat && st.dst_l->h[i].pitch == st.dst_l->h[i].width * 3 && st.dst_l->h[i].offset % 16 == 0;
        }
        st.flat = flat;
        // histogram units are 96 KB (fewer per-unit zero / merge passes);
        // pointwise units are 240 KB for LUT-only steps (each unit stages the
        // image's lane-replicated LUTs once) and 120 KB otherwise, one CTA per
        // unit so the hardware balances them (measured on the cfg2 corpus:
        // Brightness 0.334 -> 0.325 ms, Grayscale 0.339 -> 0.298 ms vs whole
        // images; persistent CTAs over 24 KB chunks were slower still)
        bool lut_only = !st.normalize && !st.stages.empty();
        for (auto& sg : st.stages) lut_only = lut_only && (sg.type == ST_LUT || sg.type == ST_EQ);
        // Equalize on flat images: one whole-image unit (lane-private histogram kernel)
        const int chunk = st.kind == SK_EQ ? (flat ? (1 << 30) : 4 * kChunk) : (lut_only ? kLutChunk : kPxChunk);
        st.unit_size = chunk;
        for (int i = 0; i < P->n; ++i) {
          if (flat) {
            const int len = sl->h[i].height * sl->h[i].width * 3;
            for (int c = 0; c * chunk < len; ++c) st.units.push_back(make_int2(i, c));
          } else {
            for (int y = 0; y < sl->h[i].height; ++y) st.units.push_back(make_int2(i, y));
          }
        }
        break;
      }
      case SK_D4: {  // 64 x 64 output tiles, unit.y = (row << 16) | col (images and masks)
        for (int i = 0; i < P->n; ++i) {
          const int H = dims[i][st.slot1].first, W = dims[i][st.slot1].second;
          for (int ty = 0; ty < (H + 63) / 64; ++ty)
            for (int tx = 0; tx < (W + 63) / 64; ++tx) st.units.push_back(make_int2(i, (ty << 16) | tx));
        }
        if (st.has_mask) st.munits = st.units;
        break;
      }
      case SK_ELASTIC:
        for (int i = 0; i < P->n; ++i) {  // strips x bands of kElBand rows, unit.y = (band << 16) | strip
          const int H = dims[i][st.slot0].first, W = dims[i][st.slot0].second;
          if ((long long)H * W >= (1ll << 30)) return fail(ALB_E_UNSUPPORTED, "ElasticTransform image >= 2^30 pixels");
          const int sw = elastic_strip(st.g_r);
          for (int ty = 0; ty < (H + kElBand - 1) / kElBand; ++ty)
            for (int tx = 0; tx < (W + sw - 1) / sw; ++tx) st.units.push_back(make_int2(i, (ty << 16) | tx));
        }
        break;
      case SK_AFFINE: {
        // 55 KB: a 64x64 tile at scale >= 0.9 needs <= (99 + 5 + 31) x (99 + 5) = 14040 words
        st.unit_size = 14080;
        for (int i = 0; i < P->n; ++i) {  // 64x64 output tiles, unit.y = (row << 16) | col
          const int H = dims[i][st.slot1].first, W = dims[i][st.slot1].second;
          for (int ty = 0; ty < (H + 63) / 64; ++ty)
            for (int tx = 0; tx < (W + 63) / 64; ++tx) st.units.push_back(make_int2(i, (ty << 16) | tx));
        }
        break;
      }
      case SK_RESAMPLE: {
        st.unit_size = kStageWords;  // 40 KB of staged window rows per band
        const alb_op& o = P->ops[st.slot0];
        if (st.interp == ALB_INTERP_BILINEAR && !st.has_mask) {
          // separable kernel: a group of G output rows needs <= ceil(G * ratio) + 1
          // new window rows (ratio = largest window/output row ratio); strips of
          // 256 output columns need <= 256 * ww / nw + 3 window columns
          int max_ww = 0;
          double ratio = 0.0, cratio = 0.0;
          for (int i = 0; i < P->n; ++i) {
            int wh = dims[i][st.slot0].first, ww = dims[i][st.slot0].second;
            if (o.kind == ALB_RANDOM_SIZED_CROP) wh = ww = std::min(o.max_side, std::min(wh, ww));
            max_ww = std::max(max_ww, ww);
            if (o.kind != ALB_GRID_DISTORTION) ratio = std::max(ratio, (double)wh / o.out_h);
          }
          if (o.kind == ALB_GRID_DISTORTION) ratio = cratio = grid_stretch(o);
          else cratio = (double)max_ww / o.out_w;
          // stage program of the step (stage_mode of stages.cuh)
          int qmode = kStagesNone;
          if (st.stages.size() == 1) {
            qmode = st.stages[0].type;
          } else if (st.stages.size() == 2) {
            const int t0 = st.stages[0].type, t1 = st.stages[1].type;
            qmode = (t0 == ST_HSV && t1 == ST_LUT) ? kStagesHsvLut : (t0 == ST_LUT && t1 == ST_HSV) ? kStagesLutHsv : -1;
          } else if (st.stages.size() > 2) {
            qmode = -1;
          }
          if (resample_q4_program_ok(qmode)) {
            // quad-column kernel: units = (image, 128-column strip, group of
            // bands of R_i rows); the window rows of a band are staged once.
            // Staged-row capacity from the budget (row tables sized for 64
            // rows); each image takes the largest band height R_i whose
            // window rows (ceil(R_i * its ratio) + 3) fit the capacity.
            const int sw = std::min(max_ww, (int)std::ceil(128.0 * cratio) + 3);
            const int nl = (qmode == ST_LUT || qmode == kStagesHsvLut || qmode == kStagesLutHsv) ? 1 : 0;
            int cap = 0;
            while (resample_q4_smem(nl, cap + 1, sw, 64, st.normalize) <= (size_t)ALB_Q4_BUDGET_KB * 1024) ++cap;
            if (cap >= 8) {
              st.rs_q = cap;
              int need = 0;  // staged rows the chosen band heights actually need
              st.rs_sw = sw;
              st.unit_rows = 64;  // row-table capacity; the band height is per unit
              st.rs_hw = ALB_Q4_BANDS;  // bands per unit
              for (int i = 0; i < P->n && st.rs_q > 0; ++i) {
                int wh = dims[i][st.slot0].first, ww = dims[i][st.slot0].second;
                if (o.kind == ALB_RANDOM_SIZED_CROP) wh = ww = std::min(o.max_side, std::min(wh, ww));
                const double ri = o.kind == ALB_GRID_DISTORTION ? ratio : (double)wh / o.out_h;
                int rc = -1;  // R_i = 4 << rc
                for (int c = ALB_Q4_MAXRC; c >= 0; --c)
                  if ((int)std::ceil((4 << c) * ri) + 3 <= cap) { rc = c; break; }
                const int H = dims[i][st.slot1].first, W = st.normalize ? P->out_w : dims[i][st.slot1].second;
                if (rc < 0 || (W + 127) / 128 > 256) { st.rs_q = 0; st.units.clear(); break; }
                need = std::max(need, (int)std::ceil((4 << rc) * ri) + 3);
                const int nb = (H + (4 << rc) - 1) / (4 << rc);
                for (int bg = 0; bg * st.rs_hw < nb; ++bg)
                  for (int x = 0, c = 0; x < W; x += 128, ++c)
                    st.units.push_back(make_int2(i, (rc << 28) | (bg << 8) | c));
              }
              if (st.rs_q > 0) {
                st.rs_q = need;  // shared memory for the rows used, not the whole budget
                break;
              }
              st.rs_hw = 0;
            }
          }
          const int sw = (std::min(max_ww, (int)std::ceil(256.0 * cratio) + 3)) | 1;
          int nl = 0;
          for (auto& sg : st.stages) nl += (sg.type == ST_LUT || sg.type == ST_EQ);
          // largest group that keeps >= 4 CTAs (16 warps) per SM, else any that fits
          for (int lim : {48 * 1024, 100 * 1024}) {  // (measured: 48 KB caps beat 30 and 20)
            for (int G : {16, 8, 4}) {
              const int ring = (int)std::ceil(G * ratio) + 2;
              if (ring > 63 || resample_sep_smem(nl, ring, sw, G, st.normalize) > (size_t)lim) continue;
              st.rs_ring = ring;
              st.rs_sw = sw;
              st.rs_hw = G;
              break;
            }
            if (st.rs_ring > 0) break;
          }
          if (st.rs_ring > 0) {
            const int R = 128;
            st.unit_rows = R;
            for (int i = 0; i < P->n; ++i) {
              const int H = dims[i][st.slot1].first, W = st.normalize ? P->out_w : dims[i][st.slot1].second;
              for (int y = 0, b = 0; y < H; y += R, ++b)
                for (int x = 0, c = 0; x < W; x += 256, ++c) st.units.push_back(make_int2(i, (b << 8) | c));
            }
            break;
          }
        }
        int R = 64;
        for (int i = 0; i < P->n; ++i) {
          if (dims[i][st.slot1].second > 2048) return fail(ALB_E_UNSUPPORTED, "resize output wider than 2048");
          int wh = dims[i][st.slot0].first, ww = dims[i][st.slot0].second;
          if (o.kind == ALB_RANDOM_SIZED_CROP) wh = ww = std::min(o.max_side, std::min(wh, ww));
          const double rows = (double)kStageWords / ww - 2.0;  // staged window rows that fit
          const double rr = o.kind == ALB_GRID_DISTORTION ? grid_stretch(o) : (double)wh / o.out_h;
          R = std::min(R, std::max(1, (int)(rows / rr)));
        }
        R = std::max(1, std::min(R, 32));
        st.unit_rows = R;
        for (int i = 0; i < P->n; ++i) {
          const int H = dims[i][st.slot1].first;
          for (int y = 0, b = 0; y < H; y += R, ++b) st.units.push_back(make_int2(i, b));
        }
        break;
      }
    }
    total_units += st.units.size() + st.munits.size();
  }
  // self-sampling pays only for few CTAs per image (every CTA draws its image's
  // params; measured: RandomCrop64 0.021 -> 0.017 ms, but the flips and the
  // pad, ~6 CTAs per image, 1-2% slower than one K0 launch)
  // (LUT steps: ~2 units of 240 KB per image; measured)
  for (auto& st : steps)
    if (st.self_sample && st.units.size() > (st.kind == SK_POINT ? 4 : 2) * (size_t)std::max(P->n, 1))
      st.self_sample = 0;
  // units are generated image by image: image i owns [ustart[i], ustart[i+1])
  for (auto& st : steps) {
    for (int pass = 0; pass < 2; ++pass) {
      const std::vector<int2>& u = pass ? st.munits : st.units;
      std::vector<int>& start = pass ? st.mstart : st.ustart;
      start.assign(P->n + 1, (int)u.size());
      for (int k = (int)u.size() - 1; k >= 0; --k) start[u[k].x] = k;
      for (int i = P->n - 1; i >= 0; --i) start[i] = std::min(start[i], start[i + 1]);
      for (size_t k = 1; k < u.size(); ++k)
        if (u[k].x < u[k - 1].x) return fail(ALB_E_CUDA, "internal: units not image-major");
    }
  }
  if (total_units) {
    std::vector<int2> all;
    all.reserve(total_units);
    for (auto& st : steps) {
      st.units_off = all.size();
      all.insert(all.end(), st.units.begin(), st.units.end());
      st.munits_off = all.size();
      all.insert(all.end(), st.munits.begin(), st.munits.end());
    }
    CUDA_TRY(cudaMalloc(&P->d_units, sizeof(int2) * all.size()));
    CUDA_TRY(cudaMemcpy(P->d_units, all.data(), sizeof(int2) * all.size(), cudaMemcpyHostToDevice));
  }
  if (n_ops > 0) {
    CUDA_TRY(cudaMalloc(&P->d_ops, sizeof(alb_op) * n_ops));
    CUDA_TRY(cudaMemcpy(P->d_ops, P->ops.data(), sizeof(alb_op) * n_ops, cudaMemcpyHostToDevice));
  }
  if (!P->gauss.empty()) {
    CUDA_TRY(cudaMalloc(&P->d_gauss, sizeof(double) * P->gauss.size()));
    CUDA_TRY(cudaMemcpy(P->d_gauss, P->gauss.data(), sizeof(double) * P->gauss.size(), cudaMemcpyHostToDevice));
  }
  // label / box work forks onto this thread's side stream: create it now, so
  // alb_apply from this thread creates nothing (checked; on failure the work
  // runs in order on the caller's stream)
  if ((mask_in || max_boxes > 0) && !side_init())
    return fail(ALB_E_CUDA, "could not create the side stream for label / box work");
  // ------------------------------------------------------------ workspace
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes, 256); return o; };
  const size_t nn = (size_t)std::max(P->n, 1);
  const size_t nops = (size_t)std::max(n_ops, 1);
  P->off_params = take(nn * nops * kMaxParams * sizeof(double));
  P->off_fired = take(nn * nops);
  P->off_dims = take(nn * (n_ops + 1) * 2 * sizeof(int32_t));
  P->off_luts = take(nn * std::max(P->n_luts, 1) * 768);
  P->off_norm = take(768 * sizeof(float));
  P->off_eqh = take(P->has_eq ? nn * 768 * sizeof(uint32_t) : 0);
  P->off_eql = take(P->has_eq ? nn * 768 : 0);
  P->off_geo = take(nn * kGeoBytes);  // per-image affine state (affine steps)
  size_t aff_units_end = 0;  // per-unit tile state of affine steps, indexed like the unit table
  for (const auto& st : steps)
    if (st.kind == SK_AFFINE) aff_units_end = std::max(aff_units_end, st.units_off + st.units.size());
  P->off_tiles = take(aff_units_end * kAffSub * kTileInfoBytes);
  for (const alb_op& o : P->ops) P->n_grid += o.kind == ALB_GRID_DISTORTION;
  P->off_grid = take(nn * P->n_grid * kGridStride * sizeof(double));  // knot displacements (R31)
  P->off_buf[0] = take(max_inter + 64);
  P->off_buf[1] = take(max_inter + 64);
  P->off_mbuf[0] = take(max_minter + 64);
  P->off_mbuf[1] = take(max_minter + 64);
  P->ws_bytes = off;
  // launches per apply (Equalize counted as the single-pass kernel when its
  // LUT pass is a packed step -- buffers 16-byte co-aligned, as torch gives)
  int L = (steps.size() == 1 && steps[0].self_sample) ? 0 : 1;  // prep
  for (size_t si = 0; si < steps.size(); ++si) {
    const PlanStep& st = steps[si];
    if (st.kind == SK_ROW || st.kind == SK_D4) {
      L += (st.has_image ? 1 : 0) + (st.has_mask ? 1 : 0);
    } else if (st.kind == SK_EQ) {
      const bool fused = si + 1 < steps.size() && steps[si + 1].kind == SK_POINT && steps[si + 1].stages.size() == 1 &&
                         !steps[si + 1].normalize && steps[si + 1].flat;
      L += fused ? 0 : 2;  // the LUT pass (the next step) is the single-pass kernel when fused
    } else if (st.kind == SK_AFFINE) {  // setup + image kernel (the raw-tap kernel gathers the labels too;
                                         // the pipelined one, ALB_AFFINE_PIPE=1, has a label kernel beside it)
      const bool generic = st.interp == ALB_INTERP_NEAREST || st.normalize || st.min_scale < 0.9f ||
                           st.unit_size < 14040;
      L += 2 + (st.has_mask && !generic && std::getenv("ALB_AFFINE_PIPE") != nullptr ? 1 : 0);
    } else {
      L += 1;
    }
  }
  if (max_boxes > 0) L += 1;
  P->n_launches = L;
  *plan_out = P.release();
  return ALB_OK;
}

void alb_plan_destroy(alb_plan* plan) { delete plan; }

alb_status alb_plan_workspace_size(const alb_plan* plan, size_t* bytes) {
  if (!plan || !bytes) return fail(ALB_E_INVALID_ARG, "null argument");
  *bytes = plan->ws_bytes;
  return ALB_OK;
}

int32_t alb_plan_num_launches(const alb_plan* plan) { return plan ? plan->n_launches : 0; }

static bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  const char* x = (const char*)a;
  const char* y = (const char*)b;
  return na && nb && x < y + nb && y < x + na;
}

alb_status alb_apply(const alb_plan* P, uint64_t seed, uint64_t first_image_index,
                     const uint8_t* img_in, uint8_t* img_out, float* out_nchw,
                     const uint8_t* mask_in, uint8_t* mask_out,
                     const float* boxes_in, const int32_t* labels_in, const int32_t* count_in,
                     float* boxes_out, int32_t* labels_out, int32_t* count_out,
                     void* workspace, size_t workspace_bytes, void* stream_) {
  if (!P) return fail(ALB_E_INVALID_ARG, "null plan");
  if (P->n == 0) return ALB_OK;
  if (!img_in) return fail(ALB_E_INVALID_ARG, "null img_in");
  const bool ends_norm = P->norm_slot >= 0;
  if (ends_norm ? !out_nchw : !img_out) return fail(ALB_E_INVALID_ARG, "null output");
  if (P->min && (!mask_in || !mask_out)) return fail(ALB_E_INVALID_ARG, "plan has masks: mask pointers required");
  if (P->max_boxes > 0 && (!boxes_in || !count_in || !boxes_out || !count_out))
    return fail(ALB_E_INVALID_ARG, "plan has boxes: box pointers required");
  if (!workspace || workspace_bytes < P->ws_bytes) return fail(ALB_E_WORKSPACE, "workspace too small");
  if (((uintptr_t)workspace & 255) != 0) return fail(ALB_E_WORKSPACE, "workspace must be 256-byte aligned");
  if (first_image_index + (uint64_t)P->n > (1ull << 32)) return fail(ALB_E_INVALID_ARG, "image index >= 2^32");
  if (!ends_norm && overlap(img_in, P->in->span, img_out, P->out->span))
    return fail(ALB_E_INVALID_ARG, "img_in and img_out overlap");
  if (ends_norm && overlap(img_in, P->in->span, out_nchw, (size_t)P->n * 3 * P->out_h * P->out_w * 4))
    return fail(ALB_E_INVALID_ARG, "img_in and out_nchw overlap");
  if (P->min && overlap(mask_in, P->min->span, mask_out, P->mout->span))
    return fail(ALB_E_INVALID_ARG, "mask_in and mask_out overlap");
  return launch_range(P, seed, first_image_index, img_in, img_out, out_nchw, mask_in, mask_out, boxes_in,
                      labels_in, count_in, boxes_out, labels_out, count_out, (uint8_t*)workspace, 0, P->n,
                      (cudaStream_t)stream_);
}

#ifndef ALB_HOST_CHUNKS
#define ALB_HOST_CHUNKS 16
#endif

alb_status alb_apply_host(const alb_plan* P, uint64_t seed, uint64_t first_image_index,
                          const uint8_t* host_in, size_t in_bytes, uint8_t* dev_in,
                          void* host_out, size_t out_bytes, void* dev_out, void* workspace,
                          size_t workspace_bytes, void* stream_) {
  if (!P || !host_in || !dev_in || !host_out || !dev_out) return fail(ALB_E_INVALID_ARG, "null argument");
  if (P->min || P->max_boxes > 0) return fail(ALB_E_UNSUPPORTED, "alb_apply_host carries images only");
  if (in_bytes < P->in->span) return fail(ALB_E_INVALID_ARG, "in_bytes smaller than the input layout");
  const bool ends_norm = P->norm_slot >= 0;
  const size_t nchw_img = (size_t)3 * P->out_h * P->out_w * 4;
  const size_t need = ends_norm ? (size_t)P->n * nchw_img : P->out->span;
  if (out_bytes < need) return fail(ALB_E_INVALID_ARG, "out_bytes smaller than the output");
  cudaStream_t stream = (cudaStream_t)stream_;
  // chunk boundaries: images in layout order with increasing, disjoint byte
  // ranges can be copied chunk by chunk, so that the H2D copy of chunk k+1,
  // the kernels of chunk k and the D2H copy of chunk k-1 overlap (two copy
  // engines + the SMs); otherwise one chunk (copy, kernels, copy)
  auto ends_in = [&](int i) {
    const alb_image_desc& d = P->in->h[i];
    return (size_t)d.offset + (size_t)(d.height - 1) * d.pitch + (size_t)d.width * 3;
  };
  auto ends_out = [&](int i) {
    if (ends_norm) return (size_t)(i + 1) * nchw_img;
    const alb_image_desc& d = P->out->h[i];
    return (size_t)d.offset + (size_t)(d.height - 1) * d.pitch + (size_t)d.width * 3;
  };
  auto start_out = [&](int i) { return ends_norm ? (size_t)i * nchw_img : (size_t)P->out->h[i].offset; };
  bool mono = P->n >= 2;
  for (int i = 1; i < P->n && mono; ++i)
    mono = (size_t)P->in->h[i].offset >= ends_in(i - 1) && start_out(i) >= ends_out(i - 1);
  const int K = mono ? std::min(P->n, ALB_HOST_CHUNKS) : 1;
  if (K > 1 && !P->s_in) {
    CUDA_TRY(cudaStreamCreateWithFlags(&P->s_in, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&P->s_out, cudaStreamNonBlocking));
  }
  while ((int)P->ev.size() < 2 * K + 2) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    P->ev.push_back(e);
  }
  uint8_t* ws = (uint8_t*)workspace;
  if (!ws || workspace_bytes < P->ws_bytes) return fail(ALB_E_WORKSPACE, "workspace too small");
  if (((uintptr_t)ws & 255) != 0) return fail(ALB_E_WORKSPACE, "workspace must be 256-byte aligned");
  if (first_image_index + (uint64_t)P->n > (1ull << 32)) return fail(ALB_E_INVALID_ARG, "image index >= 2^32");
  uint8_t* dout = ends_norm ? nullptr : (uint8_t*)dev_out;
  float* dnchw = ends_norm ? (float*)dev_out : nullptr;
  if (K == 1) {
    CUDA_TRY(cudaMemcpyAsync(dev_in, host_in, in_bytes, cudaMemcpyHostToDevice, stream));
    alb_status s = launch_range(P, seed, first_image_index, dev_in, dout, dnchw, nullptr, nullptr, nullptr,
                                nullptr, nullptr, nullptr, nullptr, nullptr, ws, 0, P->n, stream);
    if (s) return s;
    CUDA_TRY(cudaMemcpyAsync(host_out, dev_out, out_bytes, cudaMemcpyDeviceToHost, stream));
    return ALB_OK;
  }
  cudaEvent_t ev_start = P->ev[2 * K], ev_done = P->ev[2 * K + 1];
  CUDA_TRY(cudaEventRecord(ev_start, stream));  // everything earlier on the caller's stream first
  CUDA_TRY(cudaStreamWaitEvent(P->s_in, ev_start, 0));
  CUDA_TRY(cudaStreamWaitEvent(P->s_out, ev_start, 0));
  size_t in_pos = 0, out_pos = 0;
  for (int k = 0; k < K; ++k) {
    const int i0 = (int)((long long)P->n * k / K), i1 = (int)((long long)P->n * (k + 1) / K);
    const size_t in_end = k == K - 1 ? in_bytes : (size_t)P->in->h[i1].offset;
    const size_t out_end = k == K - 1 ? out_bytes : start_out(i1);
    CUDA_TRY(cudaMemcpyAsync(dev_in + in_pos, host_in + in_pos, in_end - in_pos, cudaMemcpyHostToDevice, P->s_in));
    CUDA_TRY(cudaEventRecord(P->ev[2 * k], P->s_in));
    CUDA_TRY(cudaStreamWaitEvent(stream, P->ev[2 * k], 0));
    alb_status s = launch_range(P, seed, first_image_index, dev_in, dout, dnchw, nullptr, nullptr, nullptr,
                                nullptr, nullptr, nullptr, nullptr, nullptr, ws, i0, i1, stream);
    if (s) return s;
    CUDA_TRY(cudaEventRecord(P->ev[2 * k + 1], stream));
    CUDA_TRY(cudaStreamWaitEvent(P->s_out, P->ev[2 * k + 1], 0));
    CUDA_TRY(cudaMemcpyAsync((uint8_t*)host_out + out_pos, (uint8_t*)dev_out + out_pos, out_end - out_pos,
                             cudaMemcpyDeviceToHost, P->s_out));
    in_pos = in_end;
    out_pos = out_end;
  }
  CUDA_TRY(cudaEventRecord(ev_done, P->s_out));
  CUDA_TRY(cudaStreamWaitEvent(stream, ev_done, 0));  // the caller's stream sees the whole result
  return ALB_OK;
}

alb_status alb_sample_params(const alb_pipeline* p, uint64_t seed, uint64_t first_image_index,
                             const int32_t* in_hw, int32_t n, double* params_out,
                             uint8_t* fired_out) {
  if (!p || n < 0 || (n > 0 && (!in_hw || !params_out || !fired_out)))
    return fail(ALB_E_INVALID_ARG, "null argument");
  if (n == 0) return ALB_OK;
  const int n_ops = (int)p->ops.size();
  std::vector<alb_image_desc> desc(n);
  for (int i = 0; i < n; ++i) {
    std::vector<std::pair<int, int>> dims;
    if (in_hw[2 * i] < 1 || in_hw[2 * i + 1] < 1) return fail(ALB_E_SHAPE, "image dims < 1");
    alb_status s = track_dims(p->ops, in_hw[2 * i], in_hw[2 * i + 1], dims);
    if (s) return s;
    desc[i] = alb_image_desc{0, in_hw[2 * i], in_hw[2 * i + 1], in_hw[2 * i + 1] * 3, 0};
  }
  if (n_ops == 0) return ALB_OK;
  alb_op* d_ops = nullptr;
  alb_image_desc* d_desc = nullptr;
  uint8_t* d_tab = nullptr;
  const size_t pb = (size_t)n * n_ops * kMaxParams * sizeof(double);
  const size_t fb = (size_t)n * n_ops;
  const size_t db = (size_t)n * (n_ops + 1) * 2 * sizeof(int32_t);
  alb_status st = ALB_OK;
  cudaError_t e = cudaSuccess;
  do {
    if ((e = cudaMalloc(&d_ops, sizeof(alb_op) * n_ops))) break;
    if ((e = cudaMalloc(&d_desc, sizeof(alb_image_desc) * n))) break;
    if ((e = cudaMalloc(&d_tab, pb + fb + db + 1024))) break;
    if ((e = cudaMemcpy(d_ops, p->ops.data(), sizeof(alb_op) * n_ops, cudaMemcpyHostToDevice))) break;
    if ((e = cudaMemcpy(d_desc, desc.data(), sizeof(alb_image_desc) * n, cudaMemcpyHostToDevice))) break;
    PrepArgs pa{};
    pa.ops = d_ops;
    pa.n_ops = n_ops;
    pa.n = n;
    pa.seed = seed;
    pa.first_image = (uint32_t)first_image_index;
    pa.in_desc = d_desc;
    pa.params = (double*)d_tab;
    pa.fired = d_tab + pb;
    pa.dims = (int32_t*)(d_tab + align_up(pb + fb, 256));
    pa.n_luts = 0;
    pa.norm_slot = -1;
    launch_prep(pa, 0);
    if ((e = cudaGetLastError())) break;
    if ((e = cudaMemcpy(params_out, d_tab, pb, cudaMemcpyDeviceToHost))) break;
    if ((e = cudaMemcpy(fired_out, d_tab + pb, fb, cudaMemcpyDeviceToHost))) break;
  } while (0);
  if (e != cudaSuccess) st = fail(ALB_E_CUDA, std::string("alb_sample_params: ") + cudaGetErrorString(e));
  cudaFree(d_ops);
  cudaFree(d_desc);
  cudaFree(d_tab);
  return st;
}

}  // extern "C"
