// resample.cu -- K5 Resize / RandomSizedCrop (O5/O6) with fused
// post-ops: exact flips/crops on the output coordinates, the pointwise stage
// chain (HSV / LUT / gray) and Normalize-to-fp32-NCHW output (K9, cfg4).
//
// Half-pixel bilinear: x_s = (x_d + 0.5) * ww / nw - 0.5, clamped to the
// window [0, ww-1] (replicate border at the WINDOW edge, R9).  Column and row
// tables (x0, fx, nearest) are computed in fp64 in the definition's operation
// order, so the coordinates equal the oracle's bit for bit; the blend runs in
// fp32.  Masks: nearest, round_half_up(x_s).
//
// GridDistortion (reading R31) runs through the same kernels: its source
// coordinates are separable monotone axis maps inside the image, so only the
// coordinate function changes (g_cx / g_cy, knot tables built by K0).
//
// Work unit = (image, band of `unit_rows` output rows); persistent grid over
// contiguous unit ranges; the column table is rebuilt only when the image
// changes.  Per band, the window rows it needs are staged in shared memory as
// RGBx words (16-byte loads + byte permutes).  Each warp owns output rows:
// lane = column, 4 shared-memory taps per pixel, RGB bytes into a per-warp
// shared row buffer, then the warp writes the row with aligned 16-byte stores.
#include <algorithm>

#include "stages.cuh"

namespace alb {

constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsMaxCols = 2048;
constexpr int kRsMaxBand = 64;
constexpr int kRsChunk = 512;  // output columns per row-buffer flush

struct RsGeom {
  int wx0, wy0, ww, wh;  // source window
  int nw, nh;            // resize output dims
  const double* ge;      // GridDistortion knot displacements (x at +0, y at +kGridAxis), else null
  int gn;                // GridDistortion cells per axis
};

__device__ __forceinline__ RsGeom rs_geom(const StepArgs& a, int img) {
  const alb_op& o = a.ops[a.slot0];
  RsGeom g;
  g.nw = o.out_w;
  g.nh = o.out_h;
  g.ge = nullptr;
  g.gn = 0;
  if (o.kind == ALB_GRID_DISTORTION) {  // same-size remap through the axis maps (R31)
    g.wx0 = g.wy0 = 0;
    g.nw = g.ww = dim_w(a.tab, img, a.slot0);
    g.nh = g.wh = dim_h(a.tab, img, a.slot0);
    if (fired_of(a.tab, img, a.slot0)) {  // else the same-size resize map: x_s == x_d exactly
      g.ge = grid_of(a.tab, a.ops, img, a.slot0);
      g.gn = o.num_steps;
    }
  } else if (o.kind == ALB_RANDOM_SIZED_CROP) {
    const double* q = prm_of(a.tab, img, a.slot0);
    g.ww = g.wh = (int)q[0];
    g.wx0 = (int)q[1];
    g.wy0 = (int)q[2];
  } else {
    g.wx0 = g.wy0 = 0;
    g.ww = dim_w(a.tab, img, a.slot0);
    g.wh = dim_h(a.tab, img, a.slot0);
  }
  return g;
}

// source coordinate of output index d along one axis (fp64, definition order)
__device__ __forceinline__ double rs_coord(int d, int n_src, int n_dst) {
  double s = __dsub_rn(__ddiv_rn(__dmul_rn(__dadd_rn((double)d, 0.5), (double)n_src), (double)n_dst), 0.5);
  if (s < 0.0) s = 0.0;
  if (s > (double)(n_src - 1)) s = (double)(n_src - 1);
  return s;
}

// window source column / row of output index d: the resize map, or the
// GridDistortion axis maps
__device__ __forceinline__ double g_cx(const RsGeom& g, int d) {
  return g.ge ? grid_coord(d, g.ww, g.gn, g.ge) : rs_coord(d, g.ww, g.nw);
}
__device__ __forceinline__ double g_cy(const RsGeom& g, int d) {
  return g.ge ? grid_coord(d, g.wh, g.gn, g.ge + kGridAxis) : rs_coord(d, g.wh, g.nh);
}

struct ColEnt {
  uint16_t x0, xn;  // tap-0 and nearest columns (window frame)
  float fx;
};

struct RsState {
  RsGeom g;
  Map1 m;
  int Wo, Ho;
  int sy_lo, nrows, staged, pad;
};

// kGeneric = false: bilinear, u8 output -- the uniform mode branches compile
// away (a predicated-off Normalize path would otherwise issue per pixel)
template <int kOne, bool kGeneric>
__global__ void __launch_bounds__(kRsThreads, 3) k_resample(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  StageCtx x;
  init_stages(a, x);
  ColEnt* col = reinterpret_cast<ColEnt*>(sm + x.n_lut * kLutWords);
  int* row_y0 = reinterpret_cast<int*>(col + kRsMaxCols);
  float* row_fy = reinterpret_cast<float*>(row_y0 + kRsMaxBand);
  int* row_yn = reinterpret_cast<int*>(row_fy + kRsMaxBand);
  RsState* st = reinterpret_cast<RsState*>(row_yn + kRsMaxBand);
  uint8_t* rowbuf = reinterpret_cast<uint8_t*>(st + 1) + warp * (kRsChunk * 3 + 32);
  uint32_t* stage = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(st + 1) +
                                                kRsWarps * (kRsChunk * 3 + 32));
  const bool nearest = kGeneric && a.interp == ALB_INTERP_NEAREST;
  const bool has_mask = a.mdst != nullptr;
  const bool normalize = kGeneric && a.normalize;
  const int R = a.unit_rows;

  int u0, u1;
  unit_range(a.n_units, u0, u1);
  int cur_img = -1;
  for (int u = u0; u < u1; ++u) {
    const int2 unit = a.units[u];
    const int img = unit.x;
    __syncthreads();
    if (img != cur_img) {
      load_stages(a, img, sm, x, kRsThreads);
      const RsGeom g = rs_geom(a, img);
      const int Wo = a.normalize ? a.out_w : a.ddesc[img].width;
      const int Ho = a.normalize ? a.out_h : a.ddesc[img].height;
      const Map1 m = compose_exact(a.ops, a.tab, img, a.slot0 + 1, a.slot1, Wo, Ho);
      for (int xo = threadIdx.x; xo < Wo; xo += kRsThreads) {
        const double s = g_cx(g, m.ax * xo + m.bx);
        const double f = floor(s);
        ColEnt e;
        e.x0 = (uint16_t)(int)f;
        e.xn = (uint16_t)(int)floor(__dadd_rn(s, 0.5));
        e.fx = (float)__dsub_rn(s, f);
        col[xo] = e;
      }
      if (threadIdx.x == 0) {
        st->g = g; st->m = m; st->Wo = Wo; st->Ho = Ho;
      }
      cur_img = img;
      __syncthreads();
    }
    const RsGeom g = st->g;
    const Map1 m = st->m;
    const int Wo = st->Wo, Ho = st->Ho;
    const int y0 = unit.y * R, y1 = min(Ho, y0 + R);
    if (threadIdx.x < y1 - y0) {
      const double s = g_cy(g, m.ay * (y0 + threadIdx.x) + m.by);
      const double f = floor(s);
      row_y0[threadIdx.x] = (int)f;
      row_fy[threadIdx.x] = (float)__dsub_rn(s, f);
      row_yn[threadIdx.x] = (int)floor(__dadd_rn(s, 0.5));
    }
    __syncthreads();
    // window rows this band needs (the row map is monotone)
    const int ra = row_y0[0], rb = row_y0[y1 - y0 - 1];
    const int sy_lo = min(ra, rb);
    const int nrows = min(max(ra, rb) + 1, g.wh - 1) - sy_lo + 1;
    const int S = g.ww;
    const bool staged = (long long)nrows * S <= a.unit_size;
    const alb_image_desc sd = a.sdesc[img];
    const uint8_t* wbase = a.src + sd.offset + (size_t)g.wy0 * sd.pitch + (size_t)g.wx0 * 3;
    if (staged) {
      const int per_row = (g.ww + 15) >> 4;
      const uint32_t magic = 0xffffffffu / (uint32_t)per_row + 1u;
      for (int it = threadIdx.x; it < nrows * per_row; it += kRsThreads) {
        const int r = per_row == 1 ? it : (int)__umulhi((uint32_t)it, magic);
        const int c16 = (it - r * per_row) << 4;
        const uint8_t* srow = a.src + sd.offset + (size_t)(g.wy0 + sy_lo + r) * sd.pitch;
        uint32_t w[12];
        load_window<12>(srow + (size_t)(g.wx0 + c16) * 3, srow, srow + (size_t)sd.width * 3, w);
        uint32_t* d = stage + r * S + c16;
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c16 + i < g.ww) d[i] = rgbx_of(w, i);
      }
      __syncthreads();
    }
    uint8_t* dbase = nullptr;
    int dpitch = 0;
    if (!normalize) {
      const alb_image_desc dd = a.ddesc[img];
      dbase = a.dst + dd.offset;
      dpitch = dd.pitch;
    }
    const size_t plane = (size_t)Ho * Wo;
    float* nbase = normalize ? a.nchw + (size_t)img * 3 * plane : nullptr;
    const float* nl = a.tab.norm_lut;
    for (int rr = warp; rr < y1 - y0; rr += kRsWarps) {
      const int yo = y0 + rr;
      const int ry0 = row_y0[rr];
      const int ry1 = min(ry0 + 1, g.wh - 1);
      const float fy = row_fy[rr];
      const uint32_t* p0 = stage + (ry0 - sy_lo) * S;
      const uint32_t* p1 = stage + (ry1 - sy_lo) * S;
      const uint8_t* q0 = wbase + (size_t)ry0 * sd.pitch;
      const uint8_t* q1 = wbase + (size_t)ry1 * sd.pitch;
      for (int cx0 = 0; cx0 < Wo; cx0 += kRsChunk) {
        const int cw = min(kRsChunk, Wo - cx0);
        for (int c = lane; c < cw; c += 32) {
          const int xo = cx0 + c;
          const ColEnt ce = col[xo];
          uint32_t r, gg, b;
          if (nearest) {
            const int yn = row_yn[rr];
            uint32_t t;
            if (staged) {
              t = stage[(yn - sy_lo) * S + ce.xn];
            } else {
              const uint8_t* q = wbase + (size_t)yn * sd.pitch + 3 * ce.xn;
              t = q[0] | (q[1] << 8) | (q[2] << 16);
            }
            r = t & 0xff; gg = (t >> 8) & 0xff; b = (t >> 16) & 0xff;
          } else {
            const int x0 = ce.x0, x1 = min(x0 + 1, g.ww - 1);
            uint32_t t00, t10, t01, t11;
            if (staged) {
              t00 = p0[x0]; t10 = p0[x1]; t01 = p1[x0]; t11 = p1[x1];
            } else {
              t00 = q0[3 * x0] | (q0[3 * x0 + 1] << 8) | (q0[3 * x0 + 2] << 16);
              t10 = q0[3 * x1] | (q0[3 * x1 + 1] << 8) | (q0[3 * x1 + 2] << 16);
              t01 = q1[3 * x0] | (q1[3 * x0 + 1] << 8) | (q1[3 * x0 + 2] << 16);
              t11 = q1[3 * x1] | (q1[3 * x1 + 1] << 8) | (q1[3 * x1 + 2] << 16);
            }
            bilerp3(t00, t10, t01, t11, make_float2(ce.fx, fy), r, gg, b);
            r &= 0xffu; gg &= 0xffu; b &= 0xffu;
          }
          apply_stages_t<kOne>(x, sm, lane, r, gg, b);
          if (normalize) {
            float* o = nbase + (size_t)yo * Wo + xo;
            __stcs(o, nl[r]);
            __stcs(o + plane, nl[256 + gg]);
            __stcs(o + 2 * plane, nl[512 + b]);
          } else {
            rowbuf[3 * c] = (uint8_t)r;
            rowbuf[3 * c + 1] = (uint8_t)gg;
            rowbuf[3 * c + 2] = (uint8_t)b;
          }
        }
        if (!normalize) {
          __syncwarp();
          warp_copy_row(dbase + (size_t)yo * dpitch + (size_t)cx0 * 3, rowbuf, 3 * cw, lane);
          __syncwarp();
        }
      }
      if (has_mask) {
        const alb_image_desc msd = a.msdesc[img];
        const alb_image_desc mdd = a.mddesc[img];
        const uint8_t* mrow = a.msrc + msd.offset + (size_t)(g.wy0 + row_yn[rr]) * msd.pitch + g.wx0;
        uint8_t* mo = a.mdst + mdd.offset + (size_t)yo * mdd.pitch;
        for (int xo = lane; xo < Wo; xo += 32) mo[xo] = mrow[col[xo].xn];
      }
    }
  }
}


// ============================================================ separable path
// Bilinear, no mask (Resize512, RandomSizedCrop, the fused cfg4 chain).  The
// per-channel arithmetic is bilerp3's, split at its natural seam:
//   H(r, xo) = fma(fx, p(x1, r) - p(x0, r), p(x0, r) + 0.5)    once per (window row, column)
//   V(yo, xo) = fma(fy, H(y1, xo) - H(y0, xo), H(y0, xo));  out = floor(V)
// so every output byte equals the non-separable kernel's bit for bit, while
// each horizontal lerp is shared by all output rows that use the window row.
// Work unit = (image, band of unit_rows output rows, strip of 256 columns);
// warp w owns columns [32w, 32w+32) of the strip and walks down the band in
// increasing window-row order, carrying the two current H rows in REGISTERS
// (a new H row costs two shared taps; consecutive output rows mostly reuse
// them).  Per group of G output rows:
//   1. the window rows the group newly needs arrive by TMA (cp.async.bulk,
//      one aligned row range each, issued while the previous group computes)
//      in a raw ring and are unpacked to RGBx words (16-byte aligned 16-pixel
//      runs) into a second ring; the previous group's output rows are copied
//      out (aligned 16-byte chunks of pre-shifted row buffers);
//   2. each warp forms its 32 columns of the G rows (stage chain, then u8
//      bytes into the row buffers or planar fp32 Normalize stores).
constexpr int kSepCW = 256;      // strip width (output columns) = 32 x kCols x warps
constexpr int kSepMaxG = 16;     // output rows per group
constexpr int kSepMaxBand = 128;
constexpr int kSepObp = 3 * kSepCW + 16;

struct SepRow {
  int y0, y1;  // window-frame source rows
  float fy;
  int ob;      // byte offset of the row in the output row buffers (incl. 16-byte phase)
  int yo;      // output row
  int s0, s1;  // ring slots of y0, y1
  int pad;
};
struct SepState {
  RsGeom g;
  Map1 m;
  int Wo, Ho;
};

// raw window row pitch (bytes): 16-byte aligned hull of <= sw pixels
__host__ __device__ inline int sep_raw_pitch(int sw) { return (3 * sw + 32 + 15) & ~15; }

// kCols output columns per lane: 2 for plain resamples (the per-row control
// work is shared by two pixels), 1 when a stage chain / Normalize makes each
// pixel long (more warps hide its latency)
template <int kOne, bool kNorm, int kCols>
__global__ void __launch_bounds__(256 / kCols, 3 * kCols) k_resample_sep(StepArgs a) {
  constexpr int kSepThreads = 256 / kCols;
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  StageCtx x;
  init_stages(a, x);
  const int SW = a.rs_sw, K = a.rs_ring, G = a.rs_hw;  // ring rows, staged row stride (words), group rows
  const int RP = sep_raw_pitch(SW);
  uint8_t* smb = reinterpret_cast<uint8_t*>(sm + x.n_lut * kLutWords);
  SepState* st = reinterpret_cast<SepState*>(smb);
  SepRow* rowt = reinterpret_cast<SepRow*>(smb + 128);
  uint32_t* mtab = reinterpret_cast<uint32_t*>(rowt + kSepMaxBand);   // magic_of(n), n < 64
  uint64_t* mbar = reinterpret_cast<uint64_t*>(mtab + 64);
  uint32_t* src = reinterpret_cast<uint32_t*>(mbar + 2);              // [K][SW] RGBx rows
  uint8_t* raw = reinterpret_cast<uint8_t*>(src + ((K * SW + 3) & ~3)) + 64;  // [K][RP] raw rows
  uint8_t* obuf = raw + K * RP + 64;                                  // [G][kSepObp] output rows
  // kNorm: the 3 x 256 fp32 Normalize LUT in shared memory (in place of the row buffers)
  float* nls = reinterpret_cast<float*>(obuf);
  if constexpr (kNorm) {
    for (int i = threadIdx.x; i < 768; i += kSepThreads) nls[i] = __ldg(a.tab.norm_lut + i);
  }
  const uint32_t bar = smem_u32(mbar);
  const int R = a.unit_rows;
  const uint32_t mK = magic_of((uint32_t)K);
  auto slot = [&](int r) { return r - K * fdiv(r, mK); };  // r % K, r >= 0
  if (tid < 64) mtab[tid] = magic_of((uint32_t)tid);
  if (tid == 0) mbar_init(bar);
  uint32_t parity = 0;

  int u0, u1;
  unit_range(a.n_units, u0, u1);
  int cur_img = -1;
  for (int u = u0; u < u1; ++u) {
    const int2 unit = a.units[u];
    const int img = unit.x, band = unit.y >> 8, strip = unit.y & 255;
    __syncthreads();  // previous unit fully consumed
    if (img != cur_img) {
      load_stages(a, img, sm, x, kSepThreads);
      if (tid == 0) {
        SepState s;
        s.g = rs_geom(a, img);
        s.Wo = kNorm ? a.out_w : a.ddesc[img].width;
        s.Ho = kNorm ? a.out_h : a.ddesc[img].height;
        s.m = compose_exact(a.ops, a.tab, img, a.slot0 + 1, a.slot1, s.Wo, s.Ho);
        *st = s;
      }
      cur_img = img;
      __syncthreads();
    }
    const RsGeom g = st->g;
    const Map1 m = st->m;
    const int Wo = st->Wo, Ho = st->Ho;
    const int xs0 = strip * kSepCW, cw = min(kSepCW, Wo - xs0);
    const int y0 = band * R, nr = min(R, Ho - y0);
    for (int i = tid; i < nr; i += kSepThreads) {  // i-th row in increasing source order
      const int yo = m.ay > 0 ? y0 + i : y0 + nr - 1 - i;
      const double sy = g_cy(g, m.ay * yo + m.by);
      const double f = floor(sy);
      SepRow e;
      e.y0 = (int)f;
      e.y1 = min((int)f + 1, g.wh - 1);
      e.fy = (float)__dsub_rn(sy, f);
      e.yo = yo;
      e.ob = 0;
      if constexpr (!kNorm) {
        const alb_image_desc dd = a.ddesc[img];
        e.ob = (i % G) * kSepObp + (int)((uintptr_t)(a.dst + dd.offset + (size_t)yo * dd.pitch + (size_t)xs0 * 3) & 15);
      }
      e.s0 = slot(e.y0);
      e.s1 = slot(e.y1);
      e.pad = 0;
      rowt[i] = e;
    }
    // this lane's two columns (fp64, definition order O5) and the strip's window columns
    const int cb = warp * 32 * kCols + lane;
    const int xe0 = m.ax * xs0 + m.bx, xe1 = m.ax * (xs0 + cw - 1) + m.bx;
    const int sxa = (int)floor(g_cx(g, min(xe0, xe1)));
    const int sxb = min((int)floor(g_cx(g, max(xe0, xe1))) + 1, g.ww - 1) + 1;
    int o0[kCols], o1[kCols];
    float fx[kCols];
#pragma unroll
    for (int q = 0; q < kCols; ++q) {
      const double sx = g_cx(g, m.ax * (xs0 + min(cb + 32 * q, cw - 1)) + m.bx);
      const double f = floor(sx);
      o0[q] = (int)f - sxa;
      o1[q] = min((int)f + 1, g.ww - 1) - sxa;
      fx[q] = (float)__dsub_rn(sx, f);
    }
    const alb_image_desc sd = a.sdesc[img];
    const uint8_t* wbase = a.src + sd.offset + (size_t)g.wy0 * sd.pitch;
    const int X0 = g.wx0 + sxa, X1 = g.wx0 + sxb;  // absolute source columns
    const int nrun = (X1 - X0 + 30) >> 4;
    uint8_t* gbase = nullptr;
    int dpitch = 0;
    if constexpr (!kNorm) {
      const alb_image_desc dd = a.ddesc[img];
      gbase = a.dst + dd.offset + (size_t)xs0 * 3;
      dpitch = dd.pitch;
    }
    __syncthreads();  // row table
    // TMA row copies of window rows [na, rhi] -> raw ring (thread 0)
    auto issue = [&](int na, int rhi) {
      uint32_t bytes = 0;
      for (int r = na; r <= rhi; ++r) {
        const uintptr_t row = (uintptr_t)(wbase + (size_t)r * sd.pitch);
        const uintptr_t ga = (row + 3 * X0) & ~(uintptr_t)15, gb = (row + 3 * X1 + 15) & ~(uintptr_t)15;
        bulk_g2s(smem_u32(raw + slot(r) * RP), reinterpret_cast<const void*>(ga), (uint32_t)(gb - ga), bar);
        bytes += (uint32_t)(gb - ga);
      }
      mbar_arrive_tx(bar, bytes);
    };
    auto copy_out = [&](int gi0, int ng) {  // output rows gi0 .. gi0+ng-1 (source order)
      if constexpr (!kNorm) {
        const int n = 3 * cw;
        constexpr int kFull = kSepCW * 3 / 16;
        for (int it = tid; it < ng * kFull; it += kSepThreads) {
          const int j = it / kFull, k = it - j * kFull;
          uint8_t* grow = gbase + (size_t)rowt[gi0 + j].yo * dpitch;
          const int o = (int)((uintptr_t)grow & 15);
          const int cc = ((o + 15) >> 4) + k;
          if (16 * cc + 16 <= o + n)
            __stcs(reinterpret_cast<uint4*>(grow - o + 16 * cc),
                   *reinterpret_cast<const uint4*>(obuf + j * kSepObp + 16 * cc));
        }
        for (int it = tid; it < 2 * ng; it += kSepThreads) {
          const bool head = it < ng;
          const int j = head ? it : it - ng;
          uint8_t* grow = gbase + (size_t)rowt[gi0 + j].yo * dpitch;
          const int o = (int)((uintptr_t)grow & 15);
          const uint8_t* sb = obuf + j * kSepObp;
          uint8_t* d = grow - o;
          const int e = o + n;
          if (head) {
            if (o > 0) copy_partial(d, sb, o, min(e, 16));
          } else {
            const int cc = e >> 4, hi = e & 15;
            if (hi > 0 && (cc > 0 || o == 0)) copy_partial(d + 16 * cc, sb + 16 * cc, 0, hi);
          }
        }
      }
    };
    int nxt = rowt[0].y0;  // first window row not yet staged
    if (tid == 0) issue(nxt, rowt[min(G, nr) - 1].y1);
    // this warp's current two H rows (window rows hr0, hr1), both lane columns
    float4 h0[kCols], h1[kCols];
#pragma unroll
    for (int q = 0; q < kCols; ++q) h0[q] = h1[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    int hr0 = -1, hr1 = -1;
    uint32_t a0[kCols], a1[kCols];
#pragma unroll
    for (int q = 0; q < kCols; ++q) {
      a0[q] = smem_u32(src) + 4u * (uint32_t)o0[q];
      a1[q] = smem_u32(src) + 4u * (uint32_t)o1[q];
    }
    auto hrow = [&](int sl, float4 (&h)[kCols]) {  // horizontal lerps of the staged row in slot sl
      // shared-window byte addresses: per-column bases + one row offset
      const uint32_t roff = (uint32_t)(sl * SW) * 4u;
#pragma unroll
      for (int q = 0; q < kCols; ++q) {
        uint32_t t0, t1;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(t0) : "r"(a0[q] + roff));
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(t1) : "r"(a1[q] + roff));
        constexpr uint32_t kM = 0x4B000000u;
        auto cv = [](uint32_t t, uint32_t ch) { return __uint_as_float(__byte_perm(t, kM, 0x7540u | ch)); };
        const float2 P0 = make_float2(cv(t0, 0), cv(t0, 1)), P1 = make_float2(cv(t1, 0), cv(t1, 1));
        const float2 nMh = make_float2(-8388607.5f, -8388607.5f);
        const float2 H = __ffma2_rn(make_float2(fx[q], fx[q]), __fadd2_rn(P1, make_float2(-P0.x, -P0.y)),
                                    __fadd2_rn(P0, nMh));
        const float B0 = cv(t0, 2), B1 = cv(t1, 2);
        h[q] = make_float4(H.x, H.y, fmaf(fx[q], B1 - B0, B0 + -8388607.5f), 0.f);
      }
    };
    uint8_t* olane = obuf + 3 * cb;
    int prev_gi = -1, prev_ng = 0;
    for (int gi = 0; gi < nr; gi += G) {
      const int ng = min(G, nr - gi), gl = gi + ng - 1;
      const int rhi = rowt[gl].y1;
      const int na = max(nxt, rowt[gi].y0);
      const int nn = rhi - na + 1;  // <= K
      // 1. unpack the group's new window rows; copy out the previous group
      if (nn > 0) {
        mbar_wait(bar, parity);
        parity ^= 1u;
        const uint32_t mnn = mtab[nn];
        for (int it = tid; it < nn * nrun; it += kSepThreads) {
          const int k = fdiv(it, mnn), r = na + (it - k * nn);
          const uintptr_t srow = (uintptr_t)(wbase + (size_t)r * sd.pitch);
          const int xa = (11 * (16 - (int)(srow & 15))) & 15;
          const int xs = X0 - ((X0 - xa) & 15) + 16 * k;
          if (xs >= X1) continue;
          const uintptr_t ga = (srow + 3 * X0) & ~(uintptr_t)15;
          const int sl = slot(r);
          const uint4* q = reinterpret_cast<const uint4*>(raw + sl * RP +
                                                          (int)((intptr_t)(srow + 3 * (intptr_t)xs) - (intptr_t)ga));
          uint32_t w[12];
#pragma unroll
          for (int v = 0; v < 3; ++v) {
            const uint4 z = q[v];
            w[4 * v] = z.x; w[4 * v + 1] = z.y; w[4 * v + 2] = z.z; w[4 * v + 3] = z.w;
          }
          uint32_t* d = src + sl * SW + (xs - X0);
          if (xs >= X0 && xs + 16 <= X1) {
#pragma unroll
            for (int i = 0; i < 16; ++i) d[i] = rgbx_raw(w, i);
          } else {
            const int lo_i = max(X0 - xs, 0), hi_i = min(X1 - xs, 16);
            const uint32_t vm = ((1u << hi_i) - 1u) & ~((1u << lo_i) - 1u);
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (vm & (1u << i)) d[i] = rgbx_raw(w, i);
          }
        }
        nxt = rhi + 1;
      }
      if (prev_gi >= 0) copy_out(prev_gi, prev_ng);
      __syncthreads();
      // prefetch the next group's new window rows while this group computes
      if (tid == 0 && gi + G < nr) {
        const int gl2 = min(gi + 2 * G, nr) - 1;
        const int na2 = max(nxt, rowt[gi + G].y0), rhi2 = rowt[gl2].y1;
        if (rhi2 >= na2) issue(na2, rhi2);
      }
      // 2. this warp's 32 x kCols columns of the group's output rows
      for (int j = 0; j < ng; ++j) {
        const SepRow rw = rowt[gi + j];
        if (rw.y0 != hr0) {
          if (rw.y0 == hr1) {
#pragma unroll
            for (int q = 0; q < kCols; ++q) h0[q] = h1[q];
            hr0 = hr1;
          }
          else { hrow(rw.s0, h0); hr0 = rw.y0; }
        }
        if (rw.y1 != hr1) {
          if (rw.y1 == hr0) {
#pragma unroll
            for (int q = 0; q < kCols; ++q) h1[q] = h0[q];
          }
          else hrow(rw.s1, h1);
          hr1 = rw.y1;
        }
        uint32_t rq[kCols], gq[kCols], bq[kCols];
#pragma unroll
        for (int q = 0; q < kCols; ++q) {
          const float2 V = __ffma2_rn(make_float2(rw.fy, rw.fy),
                                      __fadd2_rn(make_float2(h1[q].x, h1[q].y), make_float2(-h0[q].x, -h0[q].y)),
                                      make_float2(h0[q].x, h0[q].y));
          const float vb = fmaf(rw.fy, h1[q].z - h0[q].z, h0[q].z);
          const float2 R2 = fadd2_rm(V, make_float2(8388608.f, 8388608.f));
          rq[q] = __float_as_uint(R2.x); gq[q] = __float_as_uint(R2.y); bq[q] = __float_as_uint(__fadd_rd(vb, 8388608.f));
          if constexpr (kOne != kStagesNone || kNorm) {
            rq[q] &= 0xffu; gq[q] &= 0xffu; bq[q] &= 0xffu;
          }
        }
        if constexpr (kCols == 2) apply_stages2_t<kOne>(x, sm, lane, rq, gq, bq);
        else apply_stages_t<kOne>(x, sm, lane, rq[0], gq[0], bq[0]);
#pragma unroll
        for (int q = 0; q < kCols; ++q) {
          const uint32_t r = rq[q], gg = gq[q], b = bq[q];
          if (cb + 32 * q < cw) {
            if constexpr (kNorm) {
              const size_t plane = (size_t)Ho * Wo;
              float* o = a.nchw + (size_t)img * 3 * plane + (size_t)rw.yo * Wo + xs0 + cb + 32 * q;
              __stcs(o, nls[r]);
              __stcs(o + plane, nls[256 + gg]);
              __stcs(o + 2 * plane, nls[512 + b]);
            } else {
              uint8_t* orow = olane + rw.ob + 96 * q;
              orow[0] = (uint8_t)r;
              orow[1] = (uint8_t)gg;
              orow[2] = (uint8_t)b;
            }
          }
        }
      }
      prev_gi = gi;
      prev_ng = ng;
      __syncthreads();
    }
    copy_out(prev_gi, prev_ng);
  }
}

// ====================================================== quad-column path
// Bilinear, no mask, no fused stages (rs_q > 0).  The same separable
// arithmetic as k_resample_sep (every output byte is bit-identical to it),
// organised so that the per-pixel work is only the vertical lerp, the
// rounding and the store:
//   * work unit = (image, strip of 128 output columns, group of rs_hw bands of
//     R output rows); CTA of 4 warps.  The strip's column table (fp64,
//     definition order) is built once per unit; per band the window rows are
//     staged, then warp w walks the band's rows [wR/4, (w+1)R/4) in increasing
//     window-row order, independently of the other warps;
//   * lane l owns the 4 adjacent output columns 4l..4l+3 of the strip: its 12
//     output bytes pack into 3 words (byte permutes) and go out as 32-bit
//     stores (a warp row = 384 contiguous bytes);
//   * the band's source window rows are copied raw (RGB bytes, the 16-byte
//     aligned hull of each row) by cp.async into one of two buffers: band b + 1
//     is in flight while band b computes (one CTA walks up to ALB_Q4_BANDS
//     bands), so the global latency hides behind the arithmetic;
//   * a column's two taps are the 6 bytes at 3 x0 in a staged row: three
//     aligned 32-bit loads funnel-shifted by the row's byte phase (lane taps 12
//     bytes = 3 words apart: distinct banks);
//   * per lane the current horizontal lerps H0, H1 and D = H1 - H0 of its 4
//     columns live in registers (blue channels of column pairs on the paired
//     fp32 pipe); a new window row costs 3 loads + 2 funnel shifts + 6 byte
//     permutes + 3 paired FP ops per column.
#ifndef ALB_Q4_MINB
#define ALB_Q4_MINB 4  // CTAs per SM the register budget is sized for (128 registers, no spills; cfg4 0.325 -> 0.295 ms vs 3)
#endif
constexpr int kQThreads = 128;
constexpr int kQWarps = kQThreads / 32;
constexpr int kQCols = 128;  // strip width: 32 lanes x 4 columns

struct QRow {
  float fy;
  int s0, s1;  // window rows of the two taps (window frame)
  int yo;      // output row
};

// raw staged row pitch (bytes): the 16-byte aligned hull of a window row of
// `sw` columns (3 sw + 30 bytes) + the 3-word tap over-read, 16-byte multiple
__host__ __device__ inline int q_raw_pitch(int sw) { return ((3 * sw + 30 + 12) + 15) & ~15; }

__device__ __forceinline__ float2 f2neg(float2 v) { return make_float2(-v.x, -v.y); }

// Stage programs of the quad kernel (kOne as apply_stages_t: none, one LUT,
// HSV, gray, HSV -> LUT, LUT -> HSV) on 4 pixels, with the LUT as a compact
// 3 x 256-byte table (the CTA handles one image): same values, no lane
// replication (so the stage costs 768 bytes of shared memory, not 24 KB).
struct QStages {
  float dh, ds, dv;  // HSV stage
  int on;            // HSV / gray gate
  int hsv_first;     // HSV -> LUT (1) or LUT -> HSV (0)
};

template <int kOne>
__device__ __forceinline__ void q_stages(const QStages& q, const uint8_t* lut8, uint32_t (&r)[4], uint32_t (&g)[4],
                                         uint32_t (&b)[4]) {
  auto lut = [&]() {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      r[k] = lut8[r[k]];
      g[k] = lut8[256 + g[k]];
      b[k] = lut8[512 + b[k]];
    }
  };
  auto hsv = [&]() {
    if (!q.on) return;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t r2[2] = {r[2 * h], r[2 * h + 1]}, g2[2] = {g[2 * h], g[2 * h + 1]}, b2[2] = {b[2 * h], b[2 * h + 1]};
      hsv_shift_px2(q.dh, q.ds, q.dv, r2, g2, b2);
      r[2 * h] = r2[0]; r[2 * h + 1] = r2[1];
      g[2 * h] = g2[0]; g[2 * h + 1] = g2[1];
      b[2 * h] = b2[0]; b[2 * h + 1] = b2[1];
    }
  };
  if constexpr (kOne == ST_LUT) {
    lut();
  } else if constexpr (kOne == ST_HSV) {
    hsv();
  } else if constexpr (kOne == ST_GRAY) {
    if (q.on) {
#pragma unroll
      for (int k = 0; k < 4; ++k) r[k] = g[k] = b[k] = gray_px(r[k], g[k], b[k]);
    }
  } else if constexpr (kOne == kStagesHsvLut) {
    hsv();
    lut();
  } else if constexpr (kOne == kStagesLutHsv) {
    lut();
    hsv();
  }
}

__host__ __device__ inline bool q_stage_program_ok(int mode) {
  return mode == kStagesNone || mode == ST_LUT || mode == ST_HSV || mode == ST_GRAY || mode == kStagesHsvLut ||
         mode == kStagesLutHsv;
}

bool resample_q4_program_ok(int mode) { return q_stage_program_ok(mode); }

template <int kOne, bool kNorm>
__global__ void __launch_bounds__(kQThreads, ALB_Q4_MINB) k_resample_q4(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  const int RT = a.unit_rows, RQ = a.rs_q, RP = q_raw_pitch(a.rs_sw);
  QRow* rowt = reinterpret_cast<QRow*>(sm);                 // [2][RT] (per band, double-buffered)
  int* win = reinterpret_cast<int*>(rowt + 2 * RT);         // sxa, sxb, -, -, then [16] (sy0, nrows) per band
  float4* colt = reinterpret_cast<float4*>(win + 36);       // [128] (3 x0, fx) per column
  int* rowph = reinterpret_cast<int*>(colt + kQCols);       // [2][RQ] byte phase of each staged row
  uint8_t* raw = reinterpret_cast<uint8_t*>(rowph + ((2 * RQ + 3) & ~3));  // [2][RQ][RP] raw RGB rows (16-byte aligned)
  float* nls = reinterpret_cast<float*>(raw + 2 * (size_t)RQ * RP + 16);  // [768] (kNorm)
  uint8_t* lut8 = reinterpret_cast<uint8_t*>(nls + (kNorm ? 768 : 0));     // [768] (LUT stage)

  const int2 unit = a.units[blockIdx.x];
  // unit.y = (rc << 28) | (band group << 8) | strip; band height R = 4 << rc (planner, per image)
  const int img = unit.x, bgrp = (unit.y >> 8) & 0xfffff, strip = unit.y & 255, R = 4 << (unit.y >> 28);
  const RsGeom g = rs_geom(a, img);
  const int Wo = kNorm ? a.out_w : a.ddesc[img].width, Ho = kNorm ? a.out_h : a.ddesc[img].height;
  QStages qs{0.f, 0.f, 0.f, 0, 0};
  if constexpr (kOne != kStagesNone) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (s >= a.n_stages) break;
      const Stage st = a.stages[s];
      if (st.type == ST_LUT) {
        const uint8_t* t = a.tab.luts + ((size_t)img * a.tab.n_luts + st.lut) * 768;
        for (int i = tid; i < 192; i += kQThreads)
          reinterpret_cast<uint32_t*>(lut8)[i] = __ldg(reinterpret_cast<const uint32_t*>(t) + i);
      } else {  // HSV / gray: gate (+ params), as load_stages
        qs.on = fired_of(a.tab, img, st.slot) ? 1 : 0;
        if (st.type == ST_HSV) {
          const double* q = prm_of(a.tab, img, st.slot);
          double w = q[0] / 60.0;
          w -= 6.0 * floor(w / 6.0);
          qs.dh = (float)w;
          qs.ds = (float)q[1];
          qs.dv = (float)q[2];
          qs.hsv_first = s == 0;
        }
      }
    }
  }
  if constexpr (kNorm) {
    for (int i = tid; i < 768; i += kQThreads) nls[i] = __ldg(a.tab.norm_lut + i);
  }
  const Map1 m = compose_exact(a.ops, a.tab, img, a.slot0 + 1, a.slot1, Wo, Ho);
  const int xs0 = strip * kQCols, cw = min(kQCols, Wo - xs0);
  // column table: one strip column per thread (fp64, definition order O5)
  double csx = 0.0, cf = 0.0;
  if (tid < cw) {
    csx = g_cx(g, m.ax * (xs0 + tid) + m.bx);
    cf = floor(csx);
  }
  if (tid == 0 || tid == cw - 1) {  // the column map is monotone: the ends bound the window
    const int lo = (int)cf, hi = min((int)cf + 1, g.ww - 1) + 1;
    if (m.ax > 0) { if (tid == 0) win[0] = lo; if (tid == cw - 1) win[1] = hi; }
    else { if (tid == 0) win[1] = hi; if (tid == cw - 1) win[0] = lo; }
  }
  __syncthreads();
  const int sxa = win[0], sxb = win[1];
  if (tid < cw) {  // tap-0 byte offset in a staged row (the right tap is the next 3
    // bytes; where it is clamped to the window's last column, x1 == x0 and the
    // blend is P0 exactly, so the weight is set to 0 and the bytes read past
    // the row's data do not matter)
    const int x0 = (int)cf - sxa;
    const bool clamped = (int)cf + 1 > g.ww - 1;
    colt[tid] = make_float4(__int_as_float(3 * x0), clamped ? 0.f : (float)__dsub_rn(csx, cf), 0.f, 0.f);
  }
  const int nb_img = (Ho + R - 1) / R;
  const int b0 = bgrp * a.rs_hw, b1 = min(b0 + a.rs_hw, nb_img);
  // window rows [sy0, sy0 + nrows) of each band of the unit (first / last
  // output row in increasing window-row order, the same fp64 row coordinates
  // as the row table), once per unit
  if (tid < b1 - b0) {
    const int y0 = (b0 + tid) * R, nr = min(R, Ho - y0);
    const int yf = m.ay > 0 ? y0 : y0 + nr - 1, yl = m.ay > 0 ? y0 + nr - 1 : y0;
    const int sy0 = (int)floor(g_cy(g, m.ay * yf + m.by));
    win[4 + 2 * tid] = sy0;
    win[5 + 2 * tid] = min((int)floor(g_cy(g, m.ay * yl + m.by)) + 1, g.wh - 1) - sy0 + 1;
  }
  __syncthreads();
  // this lane's 4 columns: tap byte offsets in a staged row and weights
  uint32_t tb[4];
  float fx[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float4 e = colt[min(4 * lane + k, cw - 1)];
    tb[k] = (uint32_t)__float_as_int(e.x);
    fx[k] = e.y;
  }
  const alb_image_desc sd = a.sdesc[img];
  const int X0 = g.wx0 + sxa, X1 = g.wx0 + sxb;  // absolute source columns of the window
  const int nq = ((3 * (X1 - X0) + 30) >> 4) / 4 + 1;  // groups of 4 16-byte chunks a staged row can span
  const uint32_t mq = magic_of((uint32_t)nq);
  const uint32_t raw_a = smem_u32(raw);
  uint8_t* gbase = nullptr;
  int dpitch = 0;
  if constexpr (!kNorm) {
    const alb_image_desc dd = a.ddesc[img];
    gbase = a.dst + dd.offset + (size_t)(xs0 + 4 * lane) * 3;
    dpitch = dd.pitch;
  }
  const bool full = 4 * lane + 3 < cw;  // all 4 columns inside the strip
  const bool aligned = ((uintptr_t)gbase & 3) == 0 && (dpitch & 3) == 0;
  const int RW = (R + kQWarps - 1) / kQWarps;

  // horizontal lerps of staged row `sr` for the 4 columns:
  //   H = fma(fx, P1 - P0, P0 + 0.5)  (R, G paired per column; B paired per column pair)
  // the two taps of a column are the 6 bytes at (row data + 3 x0): three
  // aligned words, funnel-shifted by the byte phase, give u0 = R0 G0 B0 R1 and
  // u1 = G1 B1 . .
  auto hrow = [&](uint32_t rbase, float2 (&hrg)[4], float2 (&hb)[2]) {
    constexpr uint32_t kM = 0x4B000000u;
    auto cv = [](uint32_t t, uint32_t ch) { return __uint_as_float(__byte_perm(t, kM, 0x7540u | ch)); };
    const float2 nMh = make_float2(-8388607.5f, -8388607.5f);
    uint32_t u0[4], u1[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t o = rbase + tb[k], wa = o & ~3u;
      uint32_t w0, w1, w2;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w0) : "r"(wa));
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w1) : "r"(wa + 4));
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w2) : "r"(wa + 8));
      u0[k] = __funnelshift_r(w0, w1, o << 3);
      u1[k] = __funnelshift_r(w1, w2, o << 3);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 P0 = make_float2(cv(u0[k], 0), cv(u0[k], 1)), P1 = make_float2(cv(u0[k], 3), cv(u1[k], 0));
      hrg[k] = __ffma2_rn(make_float2(fx[k], fx[k]), __fadd2_rn(P1, f2neg(P0)), __fadd2_rn(P0, nMh));
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const float2 B0 = make_float2(cv(u0[2 * q], 2), cv(u0[2 * q + 1], 2));
      const float2 B1 = make_float2(cv(u1[2 * q], 1), cv(u1[2 * q + 1], 1));
      hb[q] = __ffma2_rn(make_float2(fx[2 * q], fx[2 * q + 1]), __fadd2_rn(B1, f2neg(B0)), __fadd2_rn(B0, nMh));
    }
  };
  // asynchronous copy of a band's window rows into raw buffer `bi`: row r's
  // 16-byte aligned hull of [X0, X1) lands at raw[bi][r] + 16 k; its data
  // starts at byte phase rowph[bi][r]
  auto issue = [&](int band, int bi) {
    const int sy0 = win[4 + 2 * (band - b0)], nrows = win[5 + 2 * (band - b0)];
    const uint8_t* ibase = a.src + sd.offset + (size_t)(g.wy0 + sy0) * sd.pitch + 3 * X0;
    const uint32_t rb = raw_a + (uint32_t)(bi * RQ * RP);
    // item = (row, group of 4 consecutive chunks): one address computation per 64 bytes
    for (int it = tid; it < nrows * nq; it += kQThreads) {
      const int r = fdiv(it, mq), j = it - r * nq;
      const uintptr_t g0 = (uintptr_t)(ibase + (size_t)r * sd.pitch);
      const uintptr_t ga = g0 & ~(uintptr_t)15, gb = (g0 + 3 * (X1 - X0) + 15) & ~(uintptr_t)15;
      if (j == 0) rowph[bi * RQ + r] = (int)(g0 - ga);
      const uintptr_t gs = ga + 64 * j;
      const uint32_t ds = rb + (uint32_t)(r * RP + 64 * j);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
#ifdef ALB_AB_Q4_NOSTAGE
        if (q < 0)
#else
        if (gs + 16 * q < gb)
#endif
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(ds + 16u * q), "l"(gs + 16 * q)
                       : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  issue(b0, 0);
  for (int band = b0; band < b1; ++band) {
    const int y0 = band * R, nr = min(R, Ho - y0), bi = (band - b0) & 1;
    if (band > b0) __syncthreads();  // previous band's rows and raw buffer fully consumed
    if (band + 1 < b1) issue(band + 1, bi ^ 1);  // lands while this band computes
    QRow* rt = rowt + bi * RT;
    for (int i = tid; i < nr; i += kQThreads) {  // row table in increasing window-row order
      const int yo = m.ay > 0 ? y0 + i : y0 + nr - 1 - i;
      const double sy = g_cy(g, m.ay * yo + m.by);
      const double f = floor(sy);
      QRow e;
      e.fy = (float)__dsub_rn(sy, f);
      e.s0 = (int)f;
      e.s1 = min((int)f + 1, g.wh - 1);
      e.yo = yo;
      rt[i] = e;
    }
    if (band + 1 < b1) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    const int sya = rt[0].s0;
    const uint32_t rb = raw_a + (uint32_t)(bi * RQ * RP);
    const int* ph = rowph + bi * RQ;
    auto rbase = [&](int s) { return rb + (uint32_t)((s - sya) * RP + ph[s - sya]); };
    const int i0 = warp * RW, i1 = min(i0 + RW, nr);
    // two register sets of horizontal lerps; p = 0: H0 = A, H1 = B; p = 1: H0 = B,
    // H1 = A.  Advancing by one window row refills the old H0 set (no moves).
    float2 A[4], B[4], d[4], Ab[2], Bb[2], db[2];
    int p = 0, c0 = -1, c1 = -1;  // window rows of H0 / H1
    auto emit = [&](const QRow& rw, const float2 (&h0)[4], const float2 (&hb0)[2]) {
      // V = fma(fy, D, H0); out = floor(V) (round half up: H carries the +0.5)
      const float2 fy2 = make_float2(rw.fy, rw.fy);
      const float2 mg = make_float2(8388608.f, 8388608.f);
      uint32_t rq[4], gq[4], bq[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 R2 = fadd2_rm(__ffma2_rn(fy2, d[k], h0[k]), mg);
        rq[k] = __float_as_uint(R2.x);
        gq[k] = __float_as_uint(R2.y);
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float2 B2 = fadd2_rm(__ffma2_rn(fy2, db[q], hb0[q]), mg);
        bq[2 * q] = __float_as_uint(B2.x);
        bq[2 * q + 1] = __float_as_uint(B2.y);
      }
      if constexpr (kOne != kStagesNone || kNorm) {
#pragma unroll
        for (int k = 0; k < 4; ++k) { rq[k] &= 0xffu; gq[k] &= 0xffu; bq[k] &= 0xffu; }
      }
      if constexpr (kOne != kStagesNone) q_stages<kOne>(qs, lut8, rq, gq, bq);
      if (4 * lane >= cw) return;
      if constexpr (kNorm) {  // fp32 NCHW planes: one float4 per plane when 4 columns fit
        const size_t plane = (size_t)Ho * Wo;
        float* o = a.nchw + (size_t)img * 3 * plane + (size_t)rw.yo * Wo + xs0 + 4 * lane;
        if (full && ((Wo & 3) == 0)) {
          __stcs(reinterpret_cast<float4*>(o), make_float4(nls[rq[0]], nls[rq[1]], nls[rq[2]], nls[rq[3]]));
          __stcs(reinterpret_cast<float4*>(o + plane),
                 make_float4(nls[256 + gq[0]], nls[256 + gq[1]], nls[256 + gq[2]], nls[256 + gq[3]]));
          __stcs(reinterpret_cast<float4*>(o + 2 * plane),
                 make_float4(nls[512 + bq[0]], nls[512 + bq[1]], nls[512 + bq[2]], nls[512 + bq[3]]));
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (4 * lane + k < cw) {
              __stcs(o + k, nls[rq[k]]);
              __stcs(o + plane + k, nls[256 + gq[k]]);
              __stcs(o + 2 * plane + k, nls[512 + bq[k]]);
            }
        }
        return;
      }
      uint8_t* orow = gbase + (size_t)rw.yo * dpitch;
      // R0 G0 B0 R1 | G1 B1 R2 G2 | B2 R3 G3 B3
      const uint32_t w0 = __byte_perm(__byte_perm(rq[0], gq[0], 0x0040u), __byte_perm(bq[0], rq[1], 0x0040u), 0x5410u);
      const uint32_t w1 = __byte_perm(__byte_perm(gq[1], bq[1], 0x0040u), __byte_perm(rq[2], gq[2], 0x0040u), 0x5410u);
      const uint32_t w2 = __byte_perm(__byte_perm(bq[2], rq[3], 0x0040u), __byte_perm(gq[3], bq[3], 0x0040u), 0x5410u);
#ifdef ALB_AB_Q4_NOSTORE
      if (w0 == 0x12345678u && w1 == 0x9abcdef0u && w2 == 0x0fedcba9u) *orow = 1;
      return;
#endif
      if (full && aligned) {
        uint32_t* o32 = reinterpret_cast<uint32_t*>(orow);
        __stcs(o32, w0);
        __stcs(o32 + 1, w1);
        __stcs(o32 + 2, w2);
      } else {
        const uint32_t ws[3] = {w0, w1, w2};
        const int nbytes = 3 * min(4, cw - 4 * lane);
#pragma unroll
        for (int j = 0; j < 12; ++j)
          if (j < nbytes) orow[j] = (uint8_t)(ws[j >> 2] >> (8 * (j & 3)));
      }
    };
    auto diff = [&](const float2 (&h1)[4], const float2 (&hb1)[2], const float2 (&h0)[4], const float2 (&hb0)[2]) {
#pragma unroll
      for (int k = 0; k < 4; ++k) d[k] = __fadd2_rn(h1[k], f2neg(h0[k]));  // D = H1 - H0
      db[0] = __fadd2_rn(hb1[0], f2neg(hb0[0]));
      db[1] = __fadd2_rn(hb1[1], f2neg(hb0[1]));
    };
#ifdef ALB_AB_Q4_NOCOMPUTE
    for (int i = i0; i < i0; ++i) {
#else
    for (int i = i0; i < i1; ++i) {
#endif
      const QRow rw = rt[i];
      if (rw.s0 != c0 || rw.s1 != c1) {  // warp-uniform
        if (rw.s0 == c1 && rw.s1 != rw.s0) {  // advance by one window row
          p ^= 1;
          if (p) { hrow(rbase(rw.s1), A, Ab); diff(A, Ab, B, Bb); }
          else { hrow(rbase(rw.s1), B, Bb); diff(B, Bb, A, Ab); }
        } else {
          p = 0;
          hrow(rbase(rw.s0), A, Ab);
          if (rw.s1 != rw.s0) hrow(rbase(rw.s1), B, Bb);
          else {
#pragma unroll
            for (int k = 0; k < 4; ++k) B[k] = A[k];
            Bb[0] = Ab[0]; Bb[1] = Ab[1];
          }
          diff(B, Bb, A, Ab);
        }
        c0 = rw.s0;
        c1 = rw.s1;
      }
      if (p) emit(rw, B, Bb);
      else emit(rw, A, Ab);
    }
  }
}

size_t resample_q4_smem(int n_lut_stages, int rows, int sw, int R, bool normalize) {
  // 2 row tables, window origin, column table, 2 x row phases, 2 raw row
  // buffers (+16 B over-read slack), [Normalize table], [compact LUT]
  return (size_t)2 * R * sizeof(QRow) + 144 + kQCols * 16 + (size_t)((2 * rows + 3) & ~3) * 4 +
         (size_t)2 * rows * q_raw_pitch(sw) + 16 + (normalize ? 768 * 4 : 0) + (n_lut_stages ? 768 : 0);
}

template <int kOne>
static void launch_q4_t(const StepArgs& a, size_t smem, cudaStream_t s) {
  if (a.normalize) {
    persistent_grid((const void*)k_resample_q4<kOne, true>, kQThreads, smem, a.n_units);  // smem attribute
    k_resample_q4<kOne, true><<<a.n_units, kQThreads, smem, s>>>(a);
  } else {
    persistent_grid((const void*)k_resample_q4<kOne, false>, kQThreads, smem, a.n_units);
    k_resample_q4<kOne, false><<<a.n_units, kQThreads, smem, s>>>(a);
  }
}

size_t resample_sep_smem(int n_lut_stages, int ring, int sw, int g, bool normalize) {
  return (size_t)n_lut_stages * kLutWords * 4 + 128 + kSepMaxBand * sizeof(SepRow) + 256 + 16 +
         (size_t)((ring * sw + 3) & ~3) * 4 + 64 + (size_t)ring * sep_raw_pitch(sw) + 64 +
         (normalize ? (size_t)768 * 4 : (size_t)g * kSepObp);
}

template <int kOne, bool kNorm, int kCols>
static void launch_sep_v(const StepArgs& a, size_t smem, cudaStream_t s) {
  persistent_grid((const void*)k_resample_sep<kOne, kNorm, kCols>, 256 / kCols, smem, a.n_units);  // smem attribute
  k_resample_sep<kOne, kNorm, kCols><<<a.n_units, 256 / kCols, smem, s>>>(a);  // one CTA per unit
}

template <int kOne>
static void launch_sep_t(const StepArgs& a, size_t smem, cudaStream_t s) {
  // two columns per lane (shared row control, paired-pipe stage chains),
  // except for Normalize outputs where one column per lane measured faster
  if (a.normalize) launch_sep_v<kOne, true, 1>(a, smem, s);
  else launch_sep_v<kOne, false, 2>(a, smem, s);
}

static size_t resample_smem(const StepArgs& a) {
  return (size_t)count_lut_stages(a) * kLutWords * 4 + sizeof(ColEnt) * kRsMaxCols +
         kRsMaxBand * 12 + sizeof(RsState) + kRsWarps * (kRsChunk * 3 + 32) +
         (size_t)a.unit_size * 4;
}

template <int kOne, bool kGeneric>
static void launch_resample_v(const StepArgs& a, size_t smem, cudaStream_t s) {
  const int grid = persistent_grid((const void*)k_resample<kOne, kGeneric>, kRsThreads, smem, a.n_units);
  k_resample<kOne, kGeneric><<<grid, kRsThreads, smem, s>>>(a);
}

template <int kOne>
static void launch_resample_t(const StepArgs& a, size_t smem, cudaStream_t s) {
  if (a.normalize || a.interp == ALB_INTERP_NEAREST) launch_resample_v<kOne, true>(a, smem, s);
  else launch_resample_v<kOne, false>(a, smem, s);
}

void launch_resample(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  const int mode = stage_mode(a);
  if (a.rs_q > 0) {  // quad-column path: rs_q staged window rows, rs_sw window columns per unit
    const size_t smem = resample_q4_smem(count_lut_stages(a), a.rs_q, a.rs_sw, a.unit_rows, a.normalize != 0);
    switch (mode) {  // the planner admits only these programs (q_stage_program_ok)
      case ST_LUT: launch_q4_t<ST_LUT>(a, smem, s); break;
      case ST_HSV: launch_q4_t<ST_HSV>(a, smem, s); break;
      case ST_GRAY: launch_q4_t<ST_GRAY>(a, smem, s); break;
      case kStagesHsvLut: launch_q4_t<kStagesHsvLut>(a, smem, s); break;
      case kStagesLutHsv: launch_q4_t<kStagesLutHsv>(a, smem, s); break;
      default: launch_q4_t<kStagesNone>(a, smem, s); break;
    }
    return;
  }
  if (a.rs_ring > 0) {  // separable path (planner checked capacity)
    const size_t smem = resample_sep_smem(count_lut_stages(a), a.rs_ring, a.rs_sw, a.rs_hw, a.normalize != 0);
    ALB_DISPATCH_STAGES(mode, launch_sep_t, a, smem, s)
    return;
  }
  const size_t smem = resample_smem(a);
  ALB_DISPATCH_STAGES(mode, launch_resample_t, a, smem, s)
}

}  // namespace alb
