// kernels.cuh -- launch-argument structs shared between the planner (abi.cu)
// and the sm_100a kernels.
#pragma once
#include "common.cuh"

namespace alb {

// Prep (K0): per image, draws gate + params of every slot, tracks the dims
// each slot sees, builds the composed LUT of every LUT stage and the
// Normalize LUT.
struct PrepArgs {
  const alb_op* ops;
  int32_t n_ops;
  int32_t n;
  uint64_t seed;
  uint32_t first_image;
  const alb_image_desc* in_desc;
  double* params;
  uint8_t* fired;
  int32_t* dims;
  uint8_t* luts;
  int32_t n_luts;
  int32_t lut_k0[kMaxLuts], lut_k1[kMaxLuts];
  float* norm_lut;
  int32_t norm_slot;
  int32_t img0;       // first image of this launch (CTA i -> image img0 + i)
  double* grid;       // [n][n_grid][kGridStride] (reading R31)
  int32_t n_grid;
};

// One geometric / pointwise kernel launch.
struct StepArgs {
  const uint8_t* src;
  const alb_image_desc* sdesc;
  uint8_t* dst;
  const alb_image_desc* ddesc;
  float* nchw;
  int32_t out_h, out_w;
  const uint8_t* msrc;
  const alb_image_desc* msdesc;
  uint8_t* mdst;
  const alb_image_desc* mddesc;
  const int2* units;
  int32_t n_units;
  int32_t unit_size;  // rows per unit (rowgather) / bytes per unit (flat pointwise) /
                      // shared-memory staging capacity in words (resample, affine)
  int32_t unit_rows;  // resample: output rows per unit
  int32_t slot0, slot1;
  int32_t n_stages;
  Stage stages[kMaxStages];
  int32_t normalize;
  int32_t flat;       // pointwise: 1 = whole image is one segment
  int32_t vec_ok;     // src/dst 16-byte co-aligned per segment
  int32_t channels;   // rowgather: 3 (image) or 1 (mask)
  int32_t rg_wide;    // rowgather: 1 = the step holds a crop / pad (32-pixel, 256-bit items);
                      // 2 = flips only (warp-per-row kernel, no fill)
  uint32_t fill;      // constant fill, packed RGB (pad / constant border)
  uint32_t mask_fill;
  int32_t interp, border;  // resampling op settings
  float min_scale;         // affine: smallest scale the op can draw (footprint bound)
  Tables tab;
  const alb_op* ops;
  void* geo;  // workspace scratch: per-image affine state, kGeoBytes each
  void* tiles;  // workspace scratch: per-unit affine tile state (kTileInfoBytes each), indexed like units
  int32_t img0, n_img;  // image range [img0, n_img) of this launch (per-image kernels)
  int32_t rs_ring, rs_sw, rs_hw;  // separable resample: ring rows (0 = old kernel), staged row
                                   // stride (words), output rows per group
  int32_t self_sample;             // 1: the kernel draws its images' params itself (no K0 launch)
  int32_t lut_k0, lut_k1;          // self-sampling LUT step: op slots [lut_k0, lut_k1) of its one LUT
  int32_t rs_q;                    // quad-column resample: staged window rows per unit (0 = off);
                                   // rs_sw = window columns per 128-column strip, unit_rows = R
  uint64_t seed;                   // Philox key of this apply (ElasticTransform raw planes)
  uint32_t first_image;            // global index of image 0
  const double* gauss;             // ElasticTransform: normalised weights w[0..2 g_r] (R32)
  int32_t g_r;                     // ElasticTransform kernel radius ceil(3 sigma)
  double alpha;                    // ElasticTransform displacement scale
};

constexpr int kElMaxR = 48;  // ElasticTransform radius cap (sigma <= 16, reading R32)
// shared memory of the ElasticTransform kernel for radius r (elastic.cu)
size_t elastic_smem(int r);
// output columns per ElasticTransform unit for radius r (elastic.cu)
int elastic_strip(int r);
constexpr int kElBand = 256;  // output rows per ElasticTransform unit

// shared memory of the separable resample kernel (resample.cu)
size_t resample_sep_smem(int n_lut_stages, int ring, int sw, int g, bool normalize);
// shared memory of the quad-column resample kernel: `rows` staged window rows of
// `sw` columns, R output rows per unit (resample.cu)
size_t resample_q4_smem(int n_lut_stages, int rows, int sw, int R, bool normalize);
// stage programs the quad-column kernel runs (stage_mode values)
bool resample_q4_program_ok(int mode);

constexpr int kGeoBytes = 128;
constexpr int kTileInfoBytes = 256;
// raw-tap affine kernel: output rows per CTA tile (64 = the whole 64x64 unit,
// 32 = the unit as two 64x32 halves, each its own TileInfo record)
#ifndef ALB_RT_TH
#define ALB_RT_TH 64
#endif
constexpr int kAffSub = 64 / ALB_RT_TH;  // TileInfo records per affine unit

// Equalize (R15): histogram + LUT.
struct EqArgs {
  const uint8_t* src;
  const alb_image_desc* sdesc;
  uint32_t* hist;     // [n][3][256]
  uint8_t* lut;       // [n][768]
  const int2* units;
  int32_t n_units;
  int32_t unit_size;
  int32_t n;
  int32_t img0;       // k_eq_lut: CTA i -> image img0 + i
  int32_t slot;
  Tables tab;
};

// Boxes (K11)
struct BoxArgs {
  const float* boxes_in;
  const int32_t* labels_in;
  const int32_t* count_in;
  float* boxes_out;
  int32_t* labels_out;
  int32_t* count_out;
  int32_t max_boxes;
  float min_visibility;
  int32_t n;
  Tables tab;
  const alb_op* ops;
};

// Gate + parameters of every slot of one image and the dims each slot sees
// (O1: the gate is draw 0 of its slot, always drawn;
// the params follow in the op's documented order; shape-changing ops update
// the dims only when fired).  prm [n_ops][kMaxParams], fired [n_ops], dims
// [n_ops + 1][2] (h, w).  Used by K0 (prep.cu) and, for pipelines whose only
// step is an integer geometric map, by that step's kernel itself (no K0).
__device__ __forceinline__ void sample_core(const alb_op* ops, int n_ops, uint64_t seed, uint32_t gi, int h, int w,
                                            double* prm, uint8_t* fired, int32_t* dims) {
  for (int k = 0; k < n_ops; ++k) {
    const alb_op& o = ops[k];
    double q[kMaxParams];
#pragma unroll
    for (int j = 0; j < kMaxParams; ++j) q[j] = 0.0;
    const bool f = draw_u(seed, gi, k, 0) < o.p;  // gate: draw 0, always drawn
    dims[2 * k + 0] = h;
    dims[2 * k + 1] = w;
    int nh = h, nw = w;
    switch (o.kind) {
      case ALB_ROTATE: case ALB_BRIGHTNESS: case ALB_CONTRAST: case ALB_GAMMA:
        q[0] = urange(o.lo[0], o.hi[0], draw_u(seed, gi, k, 1));
        break;
      case ALB_BRIGHTNESS_CONTRAST:
        for (int j = 0; j < 2; ++j) q[j] = urange(o.lo[j], o.hi[j], draw_u(seed, gi, k, 1 + j));
        break;
      case ALB_SHIFT_RGB: case ALB_SHIFT_HSV:
        for (int j = 0; j < 3; ++j) q[j] = urange(o.lo[j], o.hi[j], draw_u(seed, gi, k, 1 + j));
        break;
      case ALB_SHIFT_SCALE_ROTATE:
        for (int j = 0; j < 4; ++j) q[j] = urange(o.lo[j], o.hi[j], draw_u(seed, gi, k, 1 + j));
        break;
      case ALB_RANDOM_CROP:
        q[0] = (double)uint_draw(draw_u(seed, gi, k, 1), w - o.out_w + 1);
        q[1] = (double)uint_draw(draw_u(seed, gi, k, 2), h - o.out_h + 1);
        nh = o.out_h; nw = o.out_w;
        break;
      case ALB_CROP:
        q[0] = (double)o.crop_x; q[1] = (double)o.crop_y;
        nh = o.out_h; nw = o.out_w;
        break;
      case ALB_RANDOM_SIZED_CROP: {
        const int ms = h < w ? h : w;
        const int hi = o.max_side < ms ? o.max_side : ms;
        const int side = o.min_side + uint_draw(draw_u(seed, gi, k, 1), hi - o.min_side + 1);
        q[0] = (double)side;
        q[1] = (double)uint_draw(draw_u(seed, gi, k, 2), w - side + 1);
        q[2] = (double)uint_draw(draw_u(seed, gi, k, 3), h - side + 1);
        nh = o.out_h; nw = o.out_w;
        break;
      }
      case ALB_PAD_TO_SIZE: case ALB_RESIZE:
        nh = o.out_h; nw = o.out_w;
        break;
      case ALB_ROT90: case ALB_D4:  // element, uniform over the integer range
        q[0] = o.lo[0] + (double)uint_draw(draw_u(seed, gi, k, 1), (int)(o.hi[0] - o.lo[0]) + 1);
        if ((int)q[0] & 1) { nh = w; nw = h; }
        break;
      default: break;  // GridDistortion knots: K0 (prep.cu)
    }
#pragma unroll
    for (int j = 0; j < kMaxParams; ++j) prm[(size_t)k * kMaxParams + j] = q[j];
    fired[k] = f ? 1 : 0;
    if (f) { h = nh; w = nw; }
  }
  dims[2 * n_ops + 0] = h;
  dims[2 * n_ops + 1] = w;
}

// Per-image tables of ONE image in shared memory, sampled by the kernel itself
// (StepArgs::self_sample): a Tables view whose image 0 is that image.
struct SelfTables {
  double prm[kMaxOps * kMaxParams];
  uint8_t fired[kMaxOps];
  int32_t dims[2 * (kMaxOps + 1)];
};
__device__ __forceinline__ Tables self_sample_tables(const StepArgs& a, int img, SelfTables& st) {
  const alb_image_desc sd = a.channels == 3 ? a.sdesc[img] : a.msdesc[img];
  sample_core(a.ops, a.tab.n_ops, a.seed, a.first_image + (uint32_t)img, sd.height, sd.width, st.prm, st.fired,
              st.dims);
  Tables t = a.tab;
  t.params = st.prm;
  t.fired = st.fired;
  t.dims = st.dims;
  return t;
}

// one LUT op applied to channel c's value x (fp64, no contraction; K0 and the
// self-sampling LUT kernel share it, so their tables are identical)
__device__ __forceinline__ int lut_entry(int kind, const double* q, int c, int x) {
  const double v = (double)x;
  switch (kind) {
    case ALB_BRIGHTNESS: return clip_round_d(__dmul_rn(v, q[0]));
    case ALB_CONTRAST: return clip_round_d(__dadd_rn(127.5, __dmul_rn(__dsub_rn(v, 127.5), q[0])));
    case ALB_BRIGHTNESS_CONTRAST: {
      const double t = (double)clip_round_d(__dmul_rn(v, q[0]));
      return clip_round_d(__dadd_rn(127.5, __dmul_rn(__dsub_rn(t, 127.5), q[1])));
    }
    case ALB_GAMMA: return clip_round_d(__dmul_rn(255.0, pow(__ddiv_rn(v, 255.0), q[0])));
    case ALB_SHIFT_RGB: return clip_round_d(__dadd_rn(v, q[c]));
    default: return x;
  }
}

// ±1 affine integer map output -> input with a valid output rectangle.
struct Map1 {
  int ax, bx, ay, by;
  int vx0, vx1, vy0, vy1;
};

// Exact ops slots [k_begin, k_end) composed into one map from the output of
// slot k_end-1 back to the input of slot k_begin (O2-O4).  Resize
// whose input dims equal its output dims is the identity (x_s == x_d exactly).
__device__ __forceinline__ Map1 compose_exact(const alb_op* ops, const Tables& t, int img,
                                              int k_begin, int k_end, int out_w, int out_h) {
  Map1 m{1, 0, 1, 0, 0, out_w, 0, out_h};
  for (int k = k_end - 1; k >= k_begin; --k) {
    if (!fired_of(t, img, k)) continue;
    const alb_op& o = ops[k];
    const int hin = t.dims[((size_t)img * (t.n_ops + 1) + k) * 2 + 0];
    const int win = t.dims[((size_t)img * (t.n_ops + 1) + k) * 2 + 1];
    const double* q = prm_of(t, img, k);
    switch (o.kind) {
      case ALB_HFLIP: m.ax = -m.ax; m.bx = win - 1 - m.bx; break;
      case ALB_VFLIP: m.ay = -m.ay; m.by = hin - 1 - m.by; break;
      case ALB_CROP:
      case ALB_RANDOM_CROP: m.bx += (int)q[0]; m.by += (int)q[1]; break;
      case ALB_PAD_TO_SIZE: {
        const int left = (o.out_w - win) / 2, top = (o.out_h - hin) / 2;
        m.bx -= left; m.by -= top;
        int lo, hi;
        if (m.ax > 0) { lo = -m.bx; hi = win - m.bx; } else { lo = m.bx - win + 1; hi = m.bx + 1; }
        m.vx0 = max(m.vx0, lo); m.vx1 = min(m.vx1, hi);
        if (m.ay > 0) { lo = -m.by; hi = hin - m.by; } else { lo = m.by - hin + 1; hi = m.by + 1; }
        m.vy0 = max(m.vy0, lo); m.vy1 = min(m.vy1, hi);
        break;
      }
      default: break;  // identity resize
    }
  }
  return m;
}

__device__ __forceinline__ int dim_h(const Tables& t, int img, int k) {
  return t.dims[((size_t)img * (t.n_ops + 1) + k) * 2 + 0];
}
__device__ __forceinline__ int dim_w(const Tables& t, int img, int k) {
  return t.dims[((size_t)img * (t.n_ops + 1) + k) * 2 + 1];
}

// knot displacements of GridDistortion slot `slot` for image img (ordinal = GridDistortion
// slots before it)
__device__ __forceinline__ const double* grid_of(const Tables& t, const alb_op* ops, int img, int slot) {
  int g = 0;
  for (int k = 0; k < slot; ++k) g += ops[k].kind == ALB_GRID_DISTORTION;
  return t.grid + ((size_t)img * t.n_grid + g) * kGridStride;
}

// GridDistortion source coordinate of destination index x on an axis of length
// L (reading R31, operation order as DESIGN.md states it)
__device__ __forceinline__ double grid_coord(int x, int L, int n, const double* e) {
  if (L == 1) return 0.0;
  const double span = (double)(L - 1);
  const double u = __ddiv_rn(__dmul_rn((double)x, (double)n), span);
  int i = (int)floor(u);
  if (i > n - 1) i = n - 1;
  const double t = __dsub_rn(u, (double)i);
  double v = __dadd_rn((double)x, __dadd_rn(e[i], __dmul_rn(t, __dsub_rn(e[i + 1], e[i]))));
  if (v < 0.0) v = 0.0;
  if (v > span) v = span;
  return v;
}

// grid of a persistent kernel: min(n_units, SMs x occupancy), cached (launch.cu)
int persistent_grid(const void* fn, int threads, size_t smem, int n_units);
// fork / join of this (device, host thread)'s side stream: side_fork(s)
// returns a stream ordered after everything enqueued on s so far; side_join(s)
// orders s after everything enqueued on the side stream.  Work that touches
// disjoint buffers (labels vs pixels, boxes) overlaps through it.
// side_init() creates the side stream of the calling thread ahead of time
// (false if that failed: fork then returns s itself, join is a no-op).
bool side_init();
cudaStream_t side_fork(cudaStream_t s);
void side_join(cudaStream_t s);

// kernel entry points (launch helpers live next to each kernel)
void launch_prep(const PrepArgs& a, cudaStream_t s);
void launch_point(const StepArgs& a, cudaStream_t s);
// Equalize + its LUT pass in one kernel (one CTA per image; flat, co-aligned,
// the pointwise step holding only the Equalize stage)
void launch_eq_fused(const StepArgs& a, cudaStream_t s);
void launch_rowgather(const StepArgs& a, cudaStream_t s);
void launch_resample(const StepArgs& a, cudaStream_t s);
void launch_affine(const StepArgs& a, cudaStream_t s);
void launch_d4(const StepArgs& a, cudaStream_t s);
void launch_elastic(const StepArgs& a, cudaStream_t s);
void launch_eq_hist(const EqArgs& a, cudaStream_t s);
void launch_eq_lut(const EqArgs& a, cudaStream_t s);
void launch_boxes(const BoxArgs& a, cudaStream_t s);

}  // namespace alb
