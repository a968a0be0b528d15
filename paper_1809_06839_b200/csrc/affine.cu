// affine.cu -- K4 Rotate / ShiftScaleRotate (O7) with fused post
// ops (K10: RandomCrop / Crop / flips on the output coordinates), the
// pointwise stage chain, Normalize output and the nearest-neighbour mask.
//
// Inverse map per warp-output pixel (xw, yw):
//   x_s = cx + (cos*(xw-cx-tx) - sin*(yw-cy-ty)) / s,  likewise y_s,
// written as x_s = A0*xw + A1*yw + A2 with the coefficients formed in fp64.
// Coordinates: an fp64 ANCHOR per 16x16 cell of warp-output coordinates
// (split into integer + fp32 fraction) plus fp32 local offsets (<= 15 px):
//   b = fma(A0f, dxl, frac_anchor)       (per column and cell)
//   l = fma(A1f, dyl, b)                 (per pixel, both axes in one FFMA2)
// error ~4e-6 px, and a pixel's value depends only on its warp-output
// coordinates, so the fused cfg5 kernel equals the unfused kernel bit for bit.
//
// Work unit = (image, 64x64 output tile); persistent grid over contiguous
// unit ranges.  Per tile:
//  1. warp 0 derives the source footprint, the bank-friendly staged stride
//     S (= +-1 mod 32 from the rotation, so 32 consecutive output pixels hit
//     ~distinct banks: bank = (x +- y) mod 32) and the division constants;
//  2. the footprint (+ bilinear halo) is staged in shared memory as RGBx
//     words with the border resolved per staged pixel (reflect-101 or
//     constant).  Interior runs are 16 pixels whose 48 source bytes are
//     16-byte aligned (x == 11*(-rowaddr) mod 16), so three aligned vector
//     loads and one byte permute per pixel stage them; consecutive threads
//     take consecutive footprint ROWS, so their stores hit distinct banks;
//  3. each warp owns 8 output rows, lane = column (2 columns per lane):
//     paired-fp32 coordinates, magic-number floor (add.rm.f32x2), 4 shared
//     taps, paired-fp32 blend, bytes stored straight into a shared output row
//     buffer that is pre-shifted by the destination row's 16-byte phase;
//  4. the tile is copied out in 16-byte chunks that are aligned on BOTH
//     sides; the partial first / last chunk of a row is a separate item that
//     uses naturally aligned 8/4/2/1-byte pieces (no byte loops).
// Footprints larger than the staging capacity fall back to per-tap loads
// (generic variant).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "stages.cuh"

namespace alb {

constexpr int kAfThreads = 256;
constexpr int kAfWarps = kAfThreads / 32;
constexpr int kTileW = 64, kTileH = 64;
constexpr int kRowsPerWarp = kTileH / kAfWarps;
constexpr int kObPitch = 208;   // output row buffer: 15 (phase) + 3*64, rounded to 16
constexpr int kObFull = 12;     // full 16-byte chunks per output row (192 bytes)
constexpr int kMobPitch = 80;   // mask row buffer: 15 + 64, rounded to 16
constexpr int kMobFull = 4;     // full 16-byte chunks per mask row (64 bytes)
constexpr int kMStageBytes = 11264;  // staged mask footprint capacity (bytes)
constexpr float kMagic15 = 12582912.f;  // 1.5 * 2^23: floor via round-down add
constexpr uint32_t kMagic15Bits = 0x4B400000u;

struct AfCoef {
  double A[6];
};

__device__ __forceinline__ AfCoef af_coef(const StepArgs& a, int img) {
  AfCoef c;
  if (!fired_of(a.tab, img, a.slot0)) {  // gate not fired: identity map
    c.A[0] = 1; c.A[1] = 0; c.A[2] = 0; c.A[3] = 0; c.A[4] = 1; c.A[5] = 0;
    return c;
  }
  const alb_op& o = a.ops[a.slot0];
  const double* q = prm_of(a.tab, img, a.slot0);
  double dx = 0.0, dy = 0.0, s = 1.0, th;
  if (o.kind == ALB_SHIFT_SCALE_ROTATE) {
    dx = q[0]; dy = q[1]; s = q[2]; th = q[3];
  } else {
    th = q[0];
  }
  const int W = dim_w(a.tab, img, a.slot0), H = dim_h(a.tab, img, a.slot0);
  const double rad = __ddiv_rn(__dmul_rn(th, 3.141592653589793), 180.0);
  double sn, cs;
  sincos(rad, &sn, &cs);
  const double cx = __ddiv_rn((double)W - 1.0, 2.0), cy = __ddiv_rn((double)H - 1.0, 2.0);
  const double tx = __dmul_rn(dx, (double)W), ty = __dmul_rn(dy, (double)H);
  const double ux = __dadd_rn(cx, tx), uy = __dadd_rn(cy, ty);
  c.A[0] = cs / s;
  c.A[1] = -sn / s;
  c.A[2] = cx - (cs * ux - sn * uy) / s;
  c.A[3] = sn / s;
  c.A[4] = cs / s;
  c.A[5] = cy - (sn * ux + cs * uy) / s;
  return c;
}

// Per-column cell anchor: fp64 source coordinate of the cell origin, split
// into integer part (ix, iy) and fp32 fraction, plus the column's fp32 offset.
struct Anchor {
  float bx, by;  // fma(A0f, dxl, afx), fma(A3f, dxl, afy)
  int ix, iy;
};

__device__ __forceinline__ Anchor cell_anchor(const double* A, float A0f, float A3f, int xw, int cy) {
  const double xa = (double)((xw >> 4) * 16), ya = (double)(cy * 16);
  const double sx = fma(A[0], xa, fma(A[1], ya, A[2]));
  const double sy = fma(A[3], xa, fma(A[4], ya, A[5]));
  const double flx = floor(sx), fly = floor(sy);
  const float dxl = (float)(xw & 15);
  Anchor an;
  an.bx = fmaf(A0f, dxl, (float)(sx - flx));
  an.by = fmaf(A3f, dxl, (float)(sy - fly));
  an.ix = (int)flx;
  an.iy = (int)fly;
  return an;
}

struct TileGeom {
  int fx0, fy0, S, fw, fh, staged, Sm, ci0, ci1, nrun, P, pad;
  uint32_t m_fh;  // magic of fh (items are row-major across threads)
};

struct ImgState {
  double A[6];
  float Af[4];  // A0, A1, A3, A4
  Map1 m;
  int Wo, Ho, tiles_x, pad;
};

// shared-memory byte offsets (from the end of the LUT stages)
constexpr int kOffIs = 0;
constexpr int kOffTg = (int)(sizeof(ImgState) + 15) / 16 * 16;
constexpr int kOffOb = kOffTg + (int)(sizeof(TileGeom) + 15) / 16 * 16;
constexpr int kOffStage = kOffOb + kTileH * kObPitch + 16;  // 16 B slack before the stage
// after the stage (a.unit_size words + 16 B slack): mask row buffer, mask stage

// kMode: 0 = fast (bilinear image, u8 output, always staged),
//        1 = generic (runtime nearest / Normalize / unstaged fallback)
template <int kOne, bool kMask, int kMode>
__global__ void __launch_bounds__(kAfThreads, kMask ? 2 : 3) k_affine(StepArgs a) {
  extern __shared__ uint32_t sm[];
  constexpr bool kGeneric = kMode == 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  StageCtx x;
  init_stages(a, x);
  uint8_t* smb = reinterpret_cast<uint8_t*>(sm + x.n_lut * kLutWords);
  ImgState* is = reinterpret_cast<ImgState*>(smb + kOffIs);
  TileGeom* tg = reinterpret_cast<TileGeom*>(smb + kOffTg);
  uint8_t* obuf = smb + kOffOb;
  uint32_t* stage = reinterpret_cast<uint32_t*>(smb + kOffStage);
  uint8_t* mobuf = reinterpret_cast<uint8_t*>(stage + a.unit_size) + 16;
  uint8_t* mstage = mobuf + kTileH * kMobPitch;
  const bool reflect = a.border == ALB_BORDER_REFLECT_101;
  const bool nearest = kGeneric && a.interp == ALB_INTERP_NEAREST;
  const bool normalize = kGeneric && a.normalize;

  int u0, u1;
  unit_range(a.n_units, u0, u1);
  int cur_img = -1;
  for (int u = u0; u < u1; ++u) {
    const int2 unit = a.units[u];
    const int img = unit.x;
    __syncthreads();  // previous tile fully consumed
    if (img != cur_img) {
      load_stages(a, img, sm, x, kAfThreads);
      {  // per-image state precomputed by k_affine_setup (one word per thread)
        constexpr int kW = (int)sizeof(ImgState) / 4;
        if (threadIdx.x < kW)
          reinterpret_cast<uint32_t*>(is)[threadIdx.x] = __ldcg(
              reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(a.geo) + (size_t)img * kGeoBytes) +
              threadIdx.x);
      }
      cur_img = img;
      __syncthreads();
    }
    const alb_image_desc sd = a.sdesc[img];
    const int Ws = sd.width, Hs = sd.height;
    const int Wo = is->Wo, Ho = is->Ho;
    const Map1 m = is->m;
    const int tx0 = (unit.y & 0xffff) * kTileW, ty0 = (unit.y >> 16) * kTileH;
    const int tw = min(kTileW, Wo - tx0), th = min(kTileH, Ho - ty0);
    if (warp == 0) {  // tile geometry: corners on lanes 0-3
      const int xwa = m.ax * tx0 + m.bx, xwb = m.ax * (tx0 + tw - 1) + m.bx;
      const int ywa = m.ay * ty0 + m.by, ywb = m.ay * (ty0 + th - 1) + m.by;
      const double xw0 = min(xwa, xwb), xw1 = max(xwa, xwb), yw0 = min(ywa, ywb), yw1 = max(ywa, ywb);
      const double* A = is->A;
      const int c = lane & 3;
      const double xw = (c & 1) ? xw1 : xw0, yw = (c & 2) ? yw1 : yw0;
      const double sx = fma(A[0], xw, fma(A[1], yw, A[2]));
      const double sy = fma(A[3], xw, fma(A[4], yw, A[5]));
      double lx = sx, hx = sx, ly = sy, hy = sy;
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {
        lx = fmin(lx, __shfl_xor_sync(0xffffffffu, lx, o));
        hx = fmax(hx, __shfl_xor_sync(0xffffffffu, hx, o));
        ly = fmin(ly, __shfl_xor_sync(0xffffffffu, ly, o));
        hy = fmax(hy, __shfl_xor_sync(0xffffffffu, hy, o));
      }
      if (lane == 0) {
        TileGeom t;
        t.fx0 = (int)floor(lx) - 1;
        t.fy0 = (int)floor(ly) - 1;
        t.fw = (int)floor(hx) + 2 - t.fx0 + 1;
        t.fh = (int)floor(hy) + 2 - t.fy0 + 1;
        // S = +-1 mod 32: bank = (x +- y) mod 32 for staged pixel (x, y)
        const int want = fabs(A[0] + A[3]) >= fabs(A[0] - A[3]) ? 1 : 31;
        t.S = t.fw + ((want - t.fw % 32) + 32) % 32;
        t.Sm = ((t.fw + 3) >> 2) | 1;  // mask pitch = 4 * odd words
        t.Sm *= 4;
        t.staged = (long long)t.S * t.fh <= a.unit_size &&
                   (!kMask || (long long)t.Sm * t.fh <= kMStageBytes);
        t.ci0 = min(max(-t.fx0, 0), t.fw);
        t.ci1 = min(max(Ws - t.fx0, 0), t.fw);
        t.nrun = (t.ci1 - t.ci0 + 30) >> 4;
        t.P = t.ci0 + (t.fw - t.ci1);  // border columns only
        t.m_fh = magic_of((uint32_t)t.fh);
        *tg = t;
      }
    }
    __syncthreads();
    const TileGeom t = *tg;
    const uint8_t* simg = a.src + sd.offset;
    if (t.staged) {
      // pass A: interior columns, 16-pixel runs with 16-byte aligned sources;
      // thread -> (row = it % fh, run = it / fh)
      const int X0 = t.fx0 + t.ci0, X1 = t.fx0 + t.ci1;
      const int na = t.fh * t.nrun;
      for (int it = threadIdx.x; it < na; it += kAfThreads) {
        const int k = fdiv(it, t.m_fh), r = it - k * t.fh;
        bool row_in;
        const int ry = border_idx(t.fy0 + r, Hs, reflect, row_in);
        uint32_t* drow = stage + r * t.S - t.fx0;  // indexed by absolute source column
        if (!row_in) {  // constant-border row
          const int e = min(X0 + 16 * k + 16, X1);
          for (int xx = X0 + 16 * k; xx < e; ++xx) drow[xx] = a.fill;
          continue;
        }
        const uint8_t* srow = simg + (size_t)ry * sd.pitch;
        const int xa = (11 * (16 - (int)((uintptr_t)srow & 15))) & 15;
        const int xs = X0 - ((X0 - xa) & 15) + 16 * k;
        if (xs >= X1) continue;
        const uint8_t* p = srow + 3 * (ptrdiff_t)xs;  // 16-byte aligned
        const uint8_t* lo = srow + 3 * X0;
        const uint8_t* hi = srow + 3 * X1;
        uint32_t w[12];
#pragma unroll
        for (int v = 0; v < 3; ++v) {
          const uint8_t* q = p + 16 * v;
          uint4 z = make_uint4(0, 0, 0, 0);
          if (q < hi && q + 16 > lo) z = __ldg(reinterpret_cast<const uint4*>(q));
          w[4 * v] = z.x; w[4 * v + 1] = z.y; w[4 * v + 2] = z.z; w[4 * v + 3] = z.w;
        }
        uint32_t* d = drow + xs;
        if (xs >= X0 && xs + 16 <= X1) {
#pragma unroll
          for (int i = 0; i < 16; ++i) d[i] = rgbx_raw(w, i);
        } else {  // first / last run of the row: valid-pixel bit mask
          const int lo_i = max(X0 - xs, 0), hi_i = min(X1 - xs, 16);
          const uint32_t vm = ((1u << hi_i) - 1u) & ~((1u << lo_i) - 1u);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (vm & (1u << i)) d[i] = rgbx_raw(w, i);
        }
      }
      // pass B: border columns, one pixel per thread
      for (int it = threadIdx.x; it < t.fh * t.P; it += kAfThreads) {
        const int j = fdiv(it, t.m_fh), r = it - j * t.fh;
        const int c = j < t.ci0 ? j : t.ci1 + (j - t.ci0);
        bool row_in, col_in;
        const int ry = border_idx(t.fy0 + r, Hs, reflect, row_in);
        const int rx = border_idx(t.fx0 + c, Ws, reflect, col_in);
        stage[r * t.S + c] = (row_in && col_in) ? fetch_rgb(simg + (size_t)ry * sd.pitch, rx) : a.fill;
      }
      if constexpr (kMask) {
        const uint8_t* smk = a.msrc + a.msdesc[img].offset;
        const int mpitch = a.msdesc[img].pitch;
        const int X0 = t.fx0 + t.ci0, X1 = t.fx0 + t.ci1;
        const int na = t.fh * t.nrun;
        for (int it = threadIdx.x; it < na; it += kAfThreads) {
          const int k = fdiv(it, t.m_fh), r = it - k * t.fh;
          bool row_in;
          const int ry = border_idx(t.fy0 + r, Hs, reflect, row_in);
          uint8_t* drow = mstage + r * t.Sm - t.fx0;
          if (!row_in) {
            const int e = min(X0 + 16 * k + 16, X1);
            for (int xx = X0 + 16 * k; xx < e; ++xx) drow[xx] = (uint8_t)a.mask_fill;
            continue;
          }
          const uint8_t* mrow = smk + (size_t)ry * mpitch;
          const int xa = (16 - (int)((uintptr_t)mrow & 15)) & 15;
          const int xs = X0 - ((X0 - xa) & 15) + 16 * k;
          if (xs >= X1) continue;
          const uint4 z = __ldg(reinterpret_cast<const uint4*>(mrow + xs));  // intersects [X0, X1)
          const uint32_t w4[4] = {z.x, z.y, z.z, z.w};
          uint8_t* d = drow + xs;
          const int lo_i = max(X0 - xs, 0), hi_i = min(X1 - xs, 16);
          const uint32_t vm = ((1u << hi_i) - 1u) & ~((1u << lo_i) - 1u);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (vm & (1u << i)) d[i] = (uint8_t)(w4[i >> 2] >> (8 * (i & 3)));
        }
        for (int it = threadIdx.x; it < t.fh * t.P; it += kAfThreads) {
          const int j = fdiv(it, t.m_fh), r = it - j * t.fh;
          const int c = j < t.ci0 ? j : t.ci1 + (j - t.ci0);
          bool row_in, col_in;
          const int ry = border_idx(t.fy0 + r, Hs, reflect, row_in);
          const int rx = border_idx(t.fx0 + c, Ws, reflect, col_in);
          mstage[r * t.Sm + c] = (row_in && col_in) ? smk[(size_t)ry * mpitch + rx] : (uint8_t)a.mask_fill;
        }
      }
      __syncthreads();
    }
    // ---- compute: warp owns kRowsPerWarp rows; lane = columns lane, lane + 32
    const float A0f = is->Af[0], A1f = is->Af[1], A3f = is->Af[2], A4f = is->Af[3];
    const double* A = is->A;
    const float2 A14 = make_float2(A1f, A4f);
    const int ncol = tw > 32 ? 2 : 1;
    int xw[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) xw[j] = m.ax * min(tx0 + lane + 32 * j, Wo - 1) + m.bx;
    int cur_cy = -0x7fffffff;
    float2 bxy[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
    uint32_t c0[2] = {0u, 0u}, mc0[2] = {0u, 0u};
    int aix[2] = {0, 0}, aiy[2] = {0, 0};
    uint8_t* drow0 = nullptr;
    int dpitch = 0;
    if (!normalize) {
      const alb_image_desc dd = a.ddesc[img];
      drow0 = a.dst + dd.offset + (size_t)ty0 * dd.pitch + (size_t)tx0 * 3;
      dpitch = dd.pitch;
    }
    uint8_t* mrow0 = nullptr;
    int mdpitch = 0;
    if constexpr (kMask) {
      const alb_image_desc mdd = a.mddesc[img];
      mrow0 = a.mdst + mdd.offset + (size_t)ty0 * mdd.pitch + tx0;
      mdpitch = mdd.pitch;
    }
    const uint32_t* stg = stage;
    for (int i = 0; i < kRowsPerWarp; ++i) {
      const int row = warp * kRowsPerWarp + i;
      if (row >= th) break;
      const int yw = m.ay * (ty0 + row) + m.by;
      if ((yw >> 4) != cur_cy) {  // warp-uniform: fp64 anchors of this cell row
        cur_cy = yw >> 4;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (j < ncol) {
            const Anchor an = cell_anchor(A, A0f, A3f, xw[j], cur_cy);
            bxy[j] = make_float2(an.bx, an.by);
            aix[j] = an.ix; aiy[j] = an.iy;
            const int base = (an.iy - t.fy0) * t.S + (an.ix - t.fx0);
            c0[j] = (uint32_t)base - kMagic15Bits * (uint32_t)(t.S + 1);
            if constexpr (kMask) {
              const int mb = (an.iy - t.fy0) * t.Sm + (an.ix - t.fx0);
              mc0[j] = (uint32_t)mb - kMagic15Bits * (uint32_t)(t.Sm + 1);
            }
          }
        }
      }
      const float dyl = (float)(yw & 15);
      uint8_t* orow = obuf + row * kObPitch + (int)((uintptr_t)(drow0 + (size_t)row * dpitch) & 15);
      uint8_t* morow = nullptr;
      if constexpr (kMask) morow = mobuf + row * kMobPitch + (int)((uintptr_t)(mrow0 + (size_t)row * mdpitch) & 15);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (j >= ncol) break;
        const int c = lane + 32 * j;
        const float2 l = __ffma2_rn(A14, make_float2(dyl, dyl), bxy[j]);
        const float2 tq = fadd2_rm(l, make_float2(kMagic15, kMagic15));  // floor + 1.5*2^23
        const float2 fl = __fadd2_rn(tq, make_float2(-kMagic15, -kMagic15));
        const float2 fr = __fadd2_rn(l, make_float2(-fl.x, -fl.y));     // fractions
        const uint32_t qxb = __float_as_uint(tq.x), qyb = __float_as_uint(tq.y);
        uint32_t r, g, b;
        if (!kGeneric || (!nearest && t.staged)) {
          const uint32_t idx = qyb * (uint32_t)t.S + qxb + c0[j];
          const uint32_t* p0 = stg + idx;
          const uint32_t* p1 = p0 + t.S;
          bilerp3(p0[0], p0[1], p1[0], p1[1], fr, r, g, b);
        } else {
          const int qx = (int)(qxb - kMagic15Bits), qy = (int)(qyb - kMagic15Bits);
          if (nearest) {
            const int nx = qx + (fr.x >= 0.5f), ny = qy + (fr.y >= 0.5f);
            uint32_t px;
            if (t.staged) {
              px = stg[(aiy[j] + ny - t.fy0) * t.S + (aix[j] + nx - t.fx0)];
            } else {
              bool ri, ci;
              const int yy = border_idx(aiy[j] + ny, Hs, reflect, ri);
              const int xx = border_idx(aix[j] + nx, Ws, reflect, ci);
              px = (ri && ci) ? fetch_rgb(simg + (size_t)yy * sd.pitch, xx) : a.fill;
            }
            r = px & 0xff; g = (px >> 8) & 0xff; b = (px >> 16) & 0xff;
          } else {
            auto tap = [&](int px_, int py_) -> uint32_t {
              bool ri, ci;
              const int yy = border_idx(py_, Hs, reflect, ri), xx = border_idx(px_, Ws, reflect, ci);
              return (ri && ci) ? fetch_rgb(simg + (size_t)yy * sd.pitch, xx) : a.fill;
            };
            const int X = aix[j] + qx, Y = aiy[j] + qy;
            bilerp3(tap(X, Y), tap(X + 1, Y), tap(X, Y + 1), tap(X + 1, Y + 1), fr, r, g, b);
          }
        }
        if constexpr (kOne != kStagesNone) {
          r &= 0xffu; g &= 0xffu; b &= 0xffu;
          apply_stages_t<kOne>(x, sm, lane, r, g, b);
        }
        if (normalize) {
          if (c < tw) {
            const size_t plane = (size_t)Ho * Wo;
            float* o = a.nchw + (size_t)img * 3 * plane + (size_t)(ty0 + row) * Wo + tx0 + c;
            const float* nl = a.tab.norm_lut;
            __stcs(o, nl[r & 0xff]);
            __stcs(o + plane, nl[256 + (g & 0xff)]);
            __stcs(o + 2 * plane, nl[512 + (b & 0xff)]);
          }
        } else {
          orow[3 * c] = (uint8_t)r;
          orow[3 * c + 1] = (uint8_t)g;
          orow[3 * c + 2] = (uint8_t)b;
        }
        if constexpr (kMask) {
          const uint32_t nxb = qxb + (fr.x >= 0.5f ? 1u : 0u), nyb = qyb + (fr.y >= 0.5f ? 1u : 0u);
          uint8_t v;
          if (t.staged) {
            v = mstage[nyb * (uint32_t)t.Sm + nxb + mc0[j]];
          } else {
            bool ri, ci;
            const int yy = border_idx(aiy[j] + (int)(nyb - kMagic15Bits), Hs, reflect, ri);
            const int xx = border_idx(aix[j] + (int)(nxb - kMagic15Bits), Ws, reflect, ci);
            v = (ri && ci) ? a.msrc[a.msdesc[img].offset + (size_t)yy * a.msdesc[img].pitch + xx]
                           : (uint8_t)a.mask_fill;
          }
          morow[c] = v;
        }
      }
    }
    __syncthreads();
    if (!normalize)
      copy_rows_out<kObFull, kAfThreads>(drow0, dpitch, obuf, kObPitch, th, 3 * tw);
    if constexpr (kMask)
      copy_rows_out<kMobFull, kAfThreads>(mrow0, mdpitch, mobuf, kMobPitch, th, tw);
  }
}


// ===================================================== pipelined fast path
// Bilinear, no mask, u8 output, scale >= 0.9 (the single-op Rotate / SSR
// path and any fused post crop / flip).  The footprint rows of tile t+1 are
// fetched asynchronously (16-byte cp.async of each row's aligned range,
// completion on an mbarrier) into a RAW byte buffer while the CTA computes
// tile t, so no warp waits on global loads.  Warps 0-10
// compute, warp 11 is the producer.  Per tile t:
//   P: compute warps: wait raw(t); raw RGB -> RGBx stage (aligned 16-pixel
//      runs, 3 LDS.128 + 16 byte permutes); border columns; anchor table
//      (fp64 anchor per column x cell row); copy-out of tile t-1.
//      producer: geometry of tile t+1 (per-image state precomputed by
//      k_affine_setup).                                        -- barrier
//   C: compute warps: tile t, two rows x two columns per lane in flight.
//      producer: async row copies of tile t+1 into the (now free) raw buffer.
//                                                              -- barrier
constexpr int kPThreads = 384;
constexpr int kPWarps = kPThreads / 32;
constexpr int kCW = kPWarps - 1;      // compute warps
constexpr int kCThreads = kCW * 32;
constexpr int kRawPitch = 368;        // >= 3*103 + 30 bytes; pitch/16 odd (LDS.128 banks)
constexpr int kRawRows = 104;
constexpr int kRawSlack = 64;
constexpr int kPStageWords = 13416;   // S <= 129, fh <= 104 at scale >= 0.9
constexpr int kAnCells = 5;           // cell rows a 64-row tile spans

struct AnEnt {
  float bx, by;
  uint32_t c0;
  int pad;
};


struct TileCtx {
  ImgState is;
  TileGeom t;
  uint8_t* drow0;
  int img, tx0, ty0, tw, th, cy0, ncy, dpitch;
  // per footprint row r: staged columns [sx0[r], sx1[r]) (relative to fx0) --
  // the rotated tile covers only this part of the bounding box's row
  int16_t sx0[kRawRows], sx1[kRawRows];
};

static_assert(sizeof(ImgState) <= kGeoBytes, "ImgState must fit the per-image scratch");

constexpr int kPOffCtx = 0;                                            // 3 x TileCtx
constexpr int kPCtxBytes = (int)(sizeof(TileCtx) + 15) / 16 * 16;
constexpr int kPOffBar = 3 * kPCtxBytes;                               // mbarrier
constexpr int kPOffAn = kPOffBar + 16;                                 // AnEnt[kAnCells][64]
constexpr int kPOffOb = kPOffAn + kAnCells * 64 * (int)sizeof(AnEnt);  // output rows
constexpr int kPOffRaw = kPOffOb + kTileH * kObPitch + kRawSlack;      // raw rows
constexpr int kPOffStage = kPOffRaw + kRawRows * kRawPitch + kRawSlack;
constexpr int kPSmem = kPOffStage + kPStageWords * 4;

// Per-image state of the affine step (one thread per image), read by the
// producer warp whenever a tile starts a new image.
__global__ void k_affine_setup(StepArgs a) {
  const int img = a.img0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (img >= a.n_img) return;
  const AfCoef cf = af_coef(a, img);
  ImgState s;
  for (int k = 0; k < 6; ++k) s.A[k] = cf.A[k];
  s.Af[0] = (float)cf.A[0]; s.Af[1] = (float)cf.A[1];
  s.Af[2] = (float)cf.A[3]; s.Af[3] = (float)cf.A[4];
  s.Wo = a.normalize ? a.out_w : a.ddesc[img].width;
  s.Ho = a.normalize ? a.out_h : a.ddesc[img].height;
  s.m = compose_exact(a.ops, a.tab, img, a.slot0 + 1, a.slot1, s.Wo, s.Ho);
  s.tiles_x = (s.Wo + kTileW - 1) / kTileW;
  s.pad = 0;
  *reinterpret_cast<ImgState*>(reinterpret_cast<uint8_t*>(a.geo) + (size_t)img * kGeoBytes) = s;
}

// Global inputs of the producer's geometry for one unit (lane k holds word k
// of the image's ImgState).  (Loading them one tile ahead measured slower.)
struct GeomPre {
  int2 unit;
  uint32_t gw;
  int ws;
  alb_image_desc dd;
};

__device__ __forceinline__ GeomPre pipe_prefetch(const StepArgs& a, int u, int lane) {
  constexpr int kW = (int)sizeof(ImgState) / 4;
  GeomPre p;
  p.unit = __ldg(a.units + u);
  const int img = p.unit.x;
  const uint32_t* g = reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(a.geo) +
                                                        (size_t)img * kGeoBytes);
  p.gw = lane < kW ? __ldcg(g + lane) : 0u;
  p.ws = a.sdesc[img].width;
  p.dd = a.ddesc[img];
  return p;
}

// Producer warp, phase P: geometry of the prefetched unit into c.
__device__ __forceinline__ void pipe_geom(const StepArgs& a, const GeomPre& pre, TileCtx* c, const TileCtx* prev,
                                          int lane) {
  const int2 unit = pre.unit;
  const int img = unit.x;
  if (prev == nullptr || prev->img != img) {
    constexpr int kW = (int)sizeof(ImgState) / 4;
    if (lane < kW) reinterpret_cast<uint32_t*>(&c->is)[lane] = pre.gw;
  } else if (lane == 0) {
    c->is = prev->is;
  }
  __syncwarp();
  const Map1 m = c->is.m;
  const int Wo = c->is.Wo, Ho = c->is.Ho;
  const int tx0 = (unit.y & 0xffff) * kTileW, ty0 = (unit.y >> 16) * kTileH;
  const int tw = min(kTileW, Wo - tx0), th = min(kTileH, Ho - ty0);
  const int xwa = m.ax * tx0 + m.bx, xwb = m.ax * (tx0 + tw - 1) + m.bx;
  const int ywa = m.ay * ty0 + m.by, ywb = m.ay * (ty0 + th - 1) + m.by;
  const double xw0 = min(xwa, xwb), xw1 = max(xwa, xwb), yw0 = min(ywa, ywb), yw1 = max(ywa, ywb);
  const double* A = c->is.A;
  const int cc = lane & 3;
  const double xw = (cc & 1) ? xw1 : xw0, yw = (cc & 2) ? yw1 : yw0;
  const double sx = fma(A[0], xw, fma(A[1], yw, A[2]));
  const double sy = fma(A[3], xw, fma(A[4], yw, A[5]));
  double lx = sx, hx = sx, ly = sy, hy = sy;
#pragma unroll
  for (int o = 1; o <= 2; o <<= 1) {
    lx = fmin(lx, __shfl_xor_sync(0xffffffffu, lx, o));
    hx = fmax(hx, __shfl_xor_sync(0xffffffffu, hx, o));
    ly = fmin(ly, __shfl_xor_sync(0xffffffffu, ly, o));
    hy = fmax(hy, __shfl_xor_sync(0xffffffffu, hy, o));
  }
  // corners (xw0|xw1, yw0|yw1) of the tile in source space, lanes 0..3
  double vx[4], vy[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    vx[k] = __shfl_sync(0xffffffffu, sx, k);
    vy[k] = __shfl_sync(0xffffffffu, sy, k);
  }
  if (lane == 0) {
    const int Ws = pre.ws;
    TileGeom t;
    t.fx0 = (int)floor(lx) - 1;
    t.fy0 = (int)floor(ly) - 1;
    t.fw = (int)floor(hx) + 2 - t.fx0 + 1;
    t.fh = (int)floor(hy) + 2 - t.fy0 + 1;
    const int want = fabs(A[0] + A[3]) >= fabs(A[0] - A[3]) ? 1 : 31;
    t.S = t.fw + ((want - t.fw % 32) + 32) % 32;
    t.Sm = 0;
    t.staged = 1;
    t.ci0 = min(max(-t.fx0, 0), t.fw);
    t.ci1 = min(max(Ws - t.fx0, 0), t.fw);
    t.nrun = (t.ci1 - t.ci0 + 30) >> 4;
    t.P = t.ci0 + (t.fw - t.ci1);
    t.pad = 0;
    t.m_fh = magic_of((uint32_t)t.fh);
    c->t = t;
    c->img = img; c->tx0 = tx0; c->ty0 = ty0; c->tw = tw; c->th = th;
    c->cy0 = min(ywa, ywb) >> 4;
    c->ncy = (max(ywa, ywb) >> 4) - c->cy0 + 1;
    const alb_image_desc dd = pre.dd;
    c->drow0 = a.dst + dd.offset + (size_t)ty0 * dd.pitch + (size_t)tx0 * 3;
    c->dpitch = dd.pitch;
  }
  __syncwarp();
  // per-row spans: footprint row r (source row Y = fy0 + r) is tapped by the
  // output pixels whose source y lies in [Y - 1, Y + 1); their source x range
  // is the tile parallelogram cut by that strip (+ the right tap, 1 px margin).
  // fp32 with per-edge reciprocal slopes (margins cover the rounding).
  {
    const int fx0 = c->t.fx0, fy0 = c->t.fy0, fw = c->t.fw, fh = c->t.fh;
    const int ord[5] = {0, 1, 3, 2, 0};  // parallelogram vertex order
    float ex[4], ey[4], edx[4], eiy[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      ex[e] = (float)(vx[ord[e]] - fx0);
      ey[e] = (float)(vy[ord[e]] - fy0);
      edx[e] = (float)(vx[ord[e + 1]] - vx[ord[e]]);
      const float dy = (float)(vy[ord[e + 1]] - vy[ord[e]]);
      eiy[e] = dy != 0.f ? 1.f / dy : 0.f;
    }
#ifdef ALB_AB_NOSPANS
    for (int r = lane; r < fh; r += 32) { c->sx0[r] = 0; c->sx1[r] = (int16_t)fw; }
    if (fh < 0)
#endif
    for (int r = lane; r < fh; r += 32) {
      const float ya = (float)r - 1.01f, yb = (float)r + 1.01f;
      float xmn = 1e30f, xmx = -1e30f;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (ey[e] >= ya && ey[e] <= yb) { xmn = fminf(xmn, ex[e]); xmx = fmaxf(xmx, ex[e]); }
        if (eiy[e] != 0.f) {
#pragma unroll
          for (int bnd = 0; bnd < 2; ++bnd) {
            const float tt = ((bnd ? yb : ya) - ey[e]) * eiy[e];
            if (tt >= -1e-4f && tt <= 1.0001f) {
              const float xx = fmaf(tt, edx[e], ex[e]);
              xmn = fminf(xmn, xx);
              xmx = fmaxf(xmx, xx);
            }
          }
        }
      }
      int s0 = 0, s1 = 0;
      if (xmx >= xmn) {
        s0 = max((int)floorf(xmn) - 1, 0);
        s1 = min((int)floorf(xmx) + 3, fw);
        if (s1 < s0) s1 = s0;
      }
      c->sx0[r] = (int16_t)s0;
      c->sx1[r] = (int16_t)s1;
    }
  }
  __syncwarp();
}

// Producer warp, phase C: asynchronous copies of c's footprint rows, row r ->
// raw + r * kRawPitch (the 16-byte aligned hull of the row's columns).  Lane =
// row; each lane issues 16-byte cp.async (LDGSTS) copies of its rows, then one
// cp.async.mbarrier.arrive.noinc, so the mbarrier (32 expected arrivals)
// completes when every copy of the tile has landed.  Measured alternatives
// (ALB_PROF phase timing): one cp.async.bulk per row serialises the 32 lanes'
// issue (bulk copies take uniform operands) and costs 1.5x the cycles; 8 lanes
// per row (coalesced) or copies spread over all warps are slower still.
__device__ __forceinline__ void pipe_issue(const StepArgs& a, const TileCtx* c, uint8_t* raw, uint32_t bar,
                                           int lane) {
  const TileGeom t = c->t;
  const alb_image_desc sd = a.sdesc[c->img];
  const uint8_t* simg = a.src + sd.offset;
  const bool reflect = a.border == ALB_BORDER_REFLECT_101;
  {
    for (int r = lane; r < t.fh; r += 32) {
      const int X0 = t.fx0 + max((int)c->sx0[r], t.ci0), X1 = t.fx0 + min((int)c->sx1[r], t.ci1);
      if (X1 <= X0) continue;
      bool row_in;
      const int ry = border_idx(t.fy0 + r, sd.height, reflect, row_in);
      if (!row_in) continue;
      const uintptr_t g0 = (uintptr_t)(simg + (size_t)ry * sd.pitch + 3 * X0);
      const uintptr_t g1 = (uintptr_t)(simg + (size_t)ry * sd.pitch + 3 * X1);
      const uintptr_t ga = g0 & ~(uintptr_t)15, gb = (g1 + 15) & ~(uintptr_t)15;
      const uint32_t d0 = smem_u32(raw + r * kRawPitch);
#ifndef ALB_AB_NOFILL
      for (uintptr_t g = ga; g < gb; g += 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d0 + (uint32_t)(g - ga)), "l"(g)
                     : "memory");
#endif
    }
  }
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}

template <int kOne>
__global__ void __launch_bounds__(kPThreads, 2) k_affine_pipe(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool producer = warp == kPWarps - 1;
  StageCtx x;
  init_stages(a, x);
  uint8_t* smb = reinterpret_cast<uint8_t*>(sm + x.n_lut * kLutWords);
  TileCtx* ctx = reinterpret_cast<TileCtx*>(smb + kPOffCtx);
  const uint32_t bar = smem_u32(smb + kPOffBar);
  AnEnt* an = reinterpret_cast<AnEnt*>(smb + kPOffAn);
  uint8_t* obuf = smb + kPOffOb;
  uint8_t* raw = smb + kPOffRaw;
  uint32_t* stage = reinterpret_cast<uint32_t*>(smb + kPOffStage);
  const bool reflect = a.border == ALB_BORDER_REFLECT_101;

  int u0, u1;
  unit_range(a.n_units, u0, u1);
  if (u0 >= u1) return;
  if (threadIdx.x == 0) {  // one arrival per producer lane per phase (pipe_issue)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 32;\n" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (producer) {
    pipe_geom(a, pipe_prefetch(a, u0, lane), &ctx[0], nullptr, lane);
    pipe_issue(a, &ctx[0], raw, bar, lane);
  }
  __syncthreads();
  int lut_img = -1;
#ifdef ALB_PROF
  long long pr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long tq = clock64();
#endif
  for (int u = u0; u < u1; ++u) {
    const int it_t = u - u0;
    const TileCtx& c = ctx[it_t % 3];
    const TileGeom t = c.t;
    const int img = c.img;
    if (kOne != kStagesNone && img != lut_img) {
      load_stages(a, img, sm, x, kPThreads);  // LUTs are read only in phase C
      lut_img = img;
    }
    // ---------------- phase P
    if (producer) {
      if (u + 1 < u1) pipe_geom(a, pipe_prefetch(a, u + 1, lane), &ctx[(it_t + 1) % 3], &c, lane);
    } else {
      const int tid = threadIdx.x;
#ifndef ALB_AB_NOCOPYOUT
      if (it_t > 0) {  // copy-out of the previous tile
        const TileCtx& p = ctx[(it_t + 2) % 3];
        copy_rows_out<kObFull, kCThreads>(p.drow0, p.dpitch, obuf, kObPitch, p.th, 3 * p.tw);
      }
#endif
#ifdef ALB_PROF
      { const long long t1 = clock64(); pr[6] += t1 - tq; tq = t1; }
#endif
      {  // anchor table: (cell row q, column) -> fp32 offsets + tap base
        const double* A = c.is.A;
        const float A0f = c.is.Af[0], A3f = c.is.Af[2];
        const Map1 m = c.is.m;
#ifdef ALB_AB_NOANCHOR
        for (int e = tid; e < 0; e += kCThreads) {
#else
        for (int e = tid; e < 64 * c.ncy; e += kCThreads) {
#endif
          const int col = e & 63, q = e >> 6;
          const int xw = m.ax * min(c.tx0 + col, c.is.Wo - 1) + m.bx;
          const Anchor ae = cell_anchor(A, A0f, A3f, xw, c.cy0 + q);
          AnEnt en;
          en.bx = ae.bx;
          en.by = ae.by;
          // byte offset (the consumer forms 4 * index directly)
          en.c0 = 4u * ((uint32_t)((ae.iy - t.fy0) * t.S + (ae.ix - t.fx0)) - kMagic15Bits * (uint32_t)(t.S + 1));
          en.pad = 0;
          an[e] = en;
        }
      }
#ifdef ALB_PROF
      { const long long t1 = clock64(); pr[7] += t1 - tq; tq = t1; }
#endif
      const alb_image_desc sd = a.sdesc[img];
      const int Ws = sd.width, Hs = sd.height;
      const uint8_t* simg = a.src + sd.offset;
      // border columns from global (tiles at the image's left / right edge)
#ifdef ALB_AB_NOBORDER
      for (int it = tid; it < 0; it += kCThreads) {
#else
      for (int it = tid; it < t.fh * t.P; it += kCThreads) {
#endif
        const int j = fdiv(it, t.m_fh), r = it - j * t.fh;
        const int cc = j < t.ci0 ? j : t.ci1 + (j - t.ci0);
        if (cc < c.sx0[r] || cc >= c.sx1[r]) continue;
        bool row_in, col_in;
        const int ry = border_idx(t.fy0 + r, Hs, reflect, row_in);
        const int rx = border_idx(t.fx0 + cc, Ws, reflect, col_in);
        stage[r * t.S + cc] = (row_in && col_in) ? fetch_rgb(simg + (size_t)ry * sd.pitch, rx) : a.fill;
      }
#ifdef ALB_PROF
      { const long long t1 = clock64(); pr[0] += t1 - tq; tq = t1; }
#endif
      mbar_wait(bar, (uint32_t)(it_t & 1));
#ifdef ALB_PROF
      { const long long t1 = clock64(); pr[1] += t1 - tq; tq = t1; }
#endif
      // raw RGB rows -> RGBx stage; thread -> (row = it % fh, run = it / fh)
#ifdef ALB_AB_NORESTAGE
      const int na = 0;
#else
      const int na = t.fh * t.nrun;
#endif
      for (int it = tid; it < na; it += kCThreads) {
        const int k = fdiv(it, t.m_fh), r = it - k * t.fh;
        const int X0 = t.fx0 + max((int)c.sx0[r], t.ci0), X1 = t.fx0 + min((int)c.sx1[r], t.ci1);
        if (X1 <= X0) continue;
        bool row_in;
        const int ry = border_idx(t.fy0 + r, Hs, reflect, row_in);
        uint32_t* drow = stage + r * t.S - t.fx0;
        if (!row_in) {
          const int e = min(X0 + 16 * k + 16, X1);
          for (int xx = X0 + 16 * k; xx < e; ++xx) drow[xx] = a.fill;
          continue;
        }
        const uintptr_t srow = (uintptr_t)(simg + (size_t)ry * sd.pitch);
        const int xa = (11 * (16 - (int)(srow & 15))) & 15;
        const int xs = X0 - ((X0 - xa) & 15) + 16 * k;
        if (xs >= X1) continue;
        const uintptr_t ga = (srow + 3 * X0) & ~(uintptr_t)15;
        const int off = (int)((intptr_t)(srow + 3 * (intptr_t)xs) - (intptr_t)ga);  // multiple of 16
        const uint4* q = reinterpret_cast<const uint4*>(raw + r * kRawPitch + off);
        uint32_t w[12];
#pragma unroll
        for (int v = 0; v < 3; ++v) {
          const uint4 z = q[v];
          w[4 * v] = z.x; w[4 * v + 1] = z.y; w[4 * v + 2] = z.z; w[4 * v + 3] = z.w;
        }
        uint32_t* d = drow + xs;
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
    }
#ifdef ALB_PROF
    { const long long t1 = clock64(); pr[2] += t1 - tq; tq = t1; }
#endif
    __syncthreads();
#ifdef ALB_PROF
    { const long long t1 = clock64(); pr[3] += t1 - tq; tq = t1; }
#endif
    // ---------------- phase C
    if (producer) {
      if (u + 1 < u1) pipe_issue(a, &ctx[(it_t + 1) % 3], raw, bar, lane);
    } else {
      const float2 A14 = make_float2(c.is.Af[1], c.is.Af[3]);
      const uint32_t S4 = 4u * (uint32_t)t.S;  // stage row pitch in bytes
      const Map1 m = c.is.m;
      const int th = c.th, ncol = c.tw > 32 ? 2 : 1;
      const uint8_t* drow0 = c.drow0;
      const int dpitch = c.dpitch;
      // two rows (row, row + kCW) per iteration: 4 independent pixels per lane
#ifdef ALB_AB_NOCOMPUTE
      for (int r0 = warp; r0 < 0; r0 += 2 * kCW) {
#else
      for (int r0 = warp; r0 < th; r0 += 2 * kCW) {
#endif
        const bool two = r0 + kCW < th;
        float dyl[2];
        int q[2];
        uint8_t* orow[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = two || h == 0 ? r0 + h * kCW : r0;
          const int yw = m.ay * (c.ty0 + row) + m.by;
          q[h] = (yw >> 4) - c.cy0;
          dyl[h] = (float)(yw & 15);
          orow[h] = obuf + row * kObPitch + (int)((uintptr_t)(drow0 + (size_t)row * dpitch) & 15);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (j >= ncol) break;
          const int col = lane + 32 * j;
          uint32_t rr[2], gg[2], bb[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const AnEnt e = an[q[h] * 64 + col];
            const float2 l = __ffma2_rn(A14, make_float2(dyl[h], dyl[h]), make_float2(e.bx, e.by));
            const float2 tq = fadd2_rm(l, make_float2(kMagic15, kMagic15));
            const float2 fl = __fadd2_rn(tq, make_float2(-kMagic15, -kMagic15));
            const float2 fr = __fadd2_rn(l, make_float2(-fl.x, -fl.y));
            const uint32_t off = __float_as_uint(tq.y) * S4 + (__float_as_uint(tq.x) * 4u + e.c0);  // 4 * index
            const uint32_t* p0 = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(stage) + off);
            const uint32_t* p1 = reinterpret_cast<const uint32_t*>(reinterpret_cast<const char*>(stage) + (off + S4));
            bilerp3(p0[0], p0[1], p1[0], p1[1], fr, rr[h], gg[h], bb[h]);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            uint32_t r = rr[h], g = gg[h], b = bb[h];
            if constexpr (kOne != kStagesNone) {
              r &= 0xffu; g &= 0xffu; b &= 0xffu;
              apply_stages_t<kOne>(x, sm, lane, r, g, b);
            }
            if (h == 0 || two) {
              orow[h][3 * col] = (uint8_t)r;
              orow[h][3 * col + 1] = (uint8_t)g;
              orow[h][3 * col + 2] = (uint8_t)b;
            }
          }
        }
      }
    }
#ifdef ALB_PROF
    { const long long t1 = clock64(); pr[4] += t1 - tq; tq = t1; }
#endif
    __syncthreads();
#ifdef ALB_PROF
    { const long long t1 = clock64(); pr[5] += t1 - tq; tq = t1; }
#endif
  }
#ifdef ALB_PROF
  if ((blockIdx.x == 0 || blockIdx.x == 101) && lane == 0 && (warp == 0 || warp == 5 || producer))
    printf("blk %d warp %d tiles %d: copyout %lld anchor %lld border %lld mbar %lld P-post %lld barP %lld C %lld barC %lld (cycles/tile)\n",
           blockIdx.x, warp, u1 - u0, pr[6] / (u1 - u0), pr[7] / (u1 - u0), pr[0] / (u1 - u0), pr[1] / (u1 - u0), pr[2] / (u1 - u0),
           pr[3] / (u1 - u0), pr[4] / (u1 - u0), pr[5] / (u1 - u0));
#endif
  if (!producer) {
    const TileCtx& p = ctx[(u1 - 1 - u0) % 3];
    copy_rows_out<kObFull, kCThreads>(p.drow0, p.dpitch, obuf, kObPitch, p.th, 3 * p.tw);
  }
}

// ---------------------------------------------------------------------------
// k_affine_rt -- raw-tap affine kernel (the bilinear u8 fast path).
//
// One 64 x 64 output tile at a time per CTA (persistent over a contiguous
// unit range), four CTAs per SM so the phases of different CTAs overlap
// instead of an in-CTA producer pipeline.  Per tile:
//   0. (k_affine_setup_units, one thread per unit, before the kernel) the
//      tile's source footprint from its fp64 corners -> TileInfo;
//   1. footprint rows are copied RAW (RGB bytes) by 16-byte cp.async into
//      rows of pitch kRPitch, two threads per row; row r starts at
//      r * kRPitch + 16 + (its global 16-byte phase), so every copy is
//      aligned on both sides; rows outside the image are the reflect-101
//      source rows (border_idx), copied the same way; a table holds each
//      row's base (rb[r], rb[r + 1]); meanwhile the previous tile's output is
//      copied out;
//   2. border columns (x < 0 or x >= W) are filled from the reflected column
//      of the same staged row (or the fill value), one pixel per thread;
//   3. compute: warp w owns output rows [8w, 8w + 8), lane = columns lane and
//      lane + 32; the same fp64-cell-anchor / fp32-offset coordinates and the
//      same paired-fp32 blend as k_affine / k_affine_pipe (bit-identical
//      outputs), taps = 3 aligned 32-bit shared loads per tap row
//      funnel-shifted by the tap address's byte phase (no RGB -> RGBx
//      restage); bytes go to the pre-shifted output row buffer.
constexpr int kRTH = ALB_RT_TH;          // output rows per CTA tile
// measured (Rotate, cfg2 corpus): 256 threads x 1 raw buffer x 4 CTAs / SM
// 1.31 ms; two raw buffers (the next tile's copies overlapping this tile's
// compute) 512 x 2 CTAs 1.47 ms, 256 x 2 CTAs 1.48 ms; 64 x 32 half tiles
// (8 CTAs / SM) 1.32 ms
#ifndef ALB_RT_NT
#define ALB_RT_NT 256
#endif
constexpr int kRThreads = ALB_RT_NT;     // threads per CTA
#ifndef ALB_RT_TPR
#define ALB_RT_TPR 2  // threads per footprint row in the staging copies
#endif
constexpr int kRTpr = ALB_RT_TPR;
constexpr int kRWarpRows = kRTH / (kRThreads / 32);  // output rows per warp
constexpr int kRRows = kRTH == 64 ? 108 : 88;  // footprint rows (fh <= 104 / 84 at scale >= 0.9)
constexpr int kRPitch = kRTH == 64 ? 368 : 304;  // row-table layout pitch: 16 + 15 (phase) + 3 * fw + 15 (last chunk), fw <= 107 / 86;
                                                 // 92 words = -4 banks per row (a pitch of 384 = 0 banks: every row in one bank)
constexpr int kRMaxW = (kRPitch - 46) / 3;
#ifndef ALB_RT_LIN_TAN
#define ALB_RT_LIN_TAN 1e30  // linear row layout when |tan(rotation)| <= this (0: never); measured cfg2 Rotate / SSR,
                             // cfg3 Rotate: always 1.210 / 1.248 / 0.417 ms, 1.1: 1.210 / 1.248 / 0.424,
                             // never: 1.223 / 1.264 / 0.433
#endif
constexpr double kRLinTan = ALB_RT_LIN_TAN;
constexpr int kROffTab = 0;                  // int2 [kRRows]: (rb[r], rb[r + 1])
constexpr int kROffSpan = kRRows * 8;        // int [kRRows]: staged columns s0 | s1 << 16 of row r
constexpr int kROffRaw = (kRRows * 12 + 31) / 16 * 16;  // raw rows [kRRows][kRPitch]
constexpr int kRRawBytes = kRRows * (kRPitch + 16);  // raw rows: the row-table layout or a linear one (P <= kRPitch + 16)
constexpr int kRBuf = kROffRaw + kRRawBytes + 16;  // one buffer: row table + raw rows
constexpr int kRSmem = kRBuf + 2 * kTileInfoBytes;  // raw rows + two tile records (current, next)
static_assert(kRBuf % 16 == 0, "16-byte aligned buffers");
static_assert(kROffRaw % 16 == 0, "16-byte aligned raw rows");

// Everything the raw-tap kernel reads for one tile, in one record, so a CTA
// prefetches the next tile's record into shared memory with cp.async while it
// computes the current tile (no dependent global-load chain at a tile start).
struct TileInfo {
  int fx0, fy0, fw, fh;  // source footprint (bilinear halo + 1 px rounding margin)
  int img, txy, twh;     // image; tile origin tx0 | ty0 << 16; extent tw | th << 16
  uint32_t mb;           // magic of the border pass's per-row item count
  float vx[4], vy[4];    // the tile's corners in source space, relative to (fx0, fy0), parallelogram order
  double A[6];           // the image's inverse map (ImgState.A)
  float Af[4];           // A0, A1, A3, A4 in fp32
  int m_ax, m_bx, m_ay, m_by;  // fused post map (output -> warp-output coordinates)
  int Wo, Ho, Ws, Hs;          // output / source dims
  long long soff, doff;        // image offsets in the source / destination buffers
  int spitch, dpitch, Wm, Hm;  // pitches; source mask dims
  long long msoff, mdoff;      // mask offsets
  int mspitch, mdpitch;
  int P, c0;  // linear row layout (every footprint row in the image): row r at c0 + r * P, P = spitch mod 16; P = 0: row table
  float eiy[4];  // 1 / (vy[e + 1] - vy[e]) per parallelogram edge (0 for a horizontal edge), for the row spans
  int pad[4];
};
static_assert(sizeof(TileInfo) == kTileInfoBytes, "TileInfo is the per-unit scratch record");

// footprint of the output tile [tx0, tx0 + tw) x [ty0, ty0 + th) (warp-output
// coordinates through the fused post map), the bound every affine kernel uses
__device__ __forceinline__ void tile_footprint(const ImgState& s, int tx0, int ty0, int tw, int th, int& fx0,
                                               int& fy0, int& fw, int& fh, float* vx = nullptr,
                                               float* vy = nullptr) {
  const Map1& m = s.m;
  const int xwa = m.ax * tx0 + m.bx, xwb = m.ax * (tx0 + tw - 1) + m.bx;
  const int ywa = m.ay * ty0 + m.by, ywb = m.ay * (ty0 + th - 1) + m.by;
  double lx = 1e300, hx = -1e300, ly = 1e300, hy = -1e300, cx[4], cy[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double xw = (c & 1) ? max(xwa, xwb) : min(xwa, xwb);
    const double yw = (c & 2) ? max(ywa, ywb) : min(ywa, ywb);
    const double sx = fma(s.A[0], xw, fma(s.A[1], yw, s.A[2]));
    const double sy = fma(s.A[3], xw, fma(s.A[4], yw, s.A[5]));
    lx = fmin(lx, sx); hx = fmax(hx, sx); ly = fmin(ly, sy); hy = fmax(hy, sy);
    cx[c] = sx;
    cy[c] = sy;
  }
  fx0 = (int)floor(lx) - 1;
  fy0 = (int)floor(ly) - 1;
  fw = (int)floor(hx) + 2 - fx0 + 1;
  fh = (int)floor(hy) + 2 - fy0 + 1;
  if (vx != nullptr) {  // corners in parallelogram order (0, 1, 3, 2), relative to the footprint origin
    const int ord[4] = {0, 1, 3, 2};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      vx[e] = (float)(cx[ord[e]] - fx0);
      vy[e] = (float)(cy[ord[e]] - fy0);
    }
  }
}

// Columns [s0, s1) (relative to fx0) of footprint row r that the tile's
// bilinear taps can touch: the parallelogram of the tile's source points cut
// by the strip y in [r - 1, r + 1] (a source row is tapped by points within
// one row of it), widened by the right tap and a rounding margin -- the same
// fp32 construction as the pipelined kernel's per-row spans.
__device__ __forceinline__ void row_span(const TileInfo& t, int r, int& s0, int& s1) {
  const float ya = (float)r - 1.01f, yb = (float)r + 1.01f;
  float xmn = 1e30f, xmx = -1e30f;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int e1 = (e + 1) & 3;
    const float ex = t.vx[e], ey = t.vy[e];
    const float edx = t.vx[e1] - ex, eiy = t.eiy[e];
    if (ey >= ya && ey <= yb) { xmn = fminf(xmn, ex); xmx = fmaxf(xmx, ex); }
    if (eiy != 0.f) {
#pragma unroll
      for (int bnd = 0; bnd < 2; ++bnd) {
        const float tt = ((bnd ? yb : ya) - ey) * eiy;
        if (tt >= -1e-4f && tt <= 1.0001f) {
          const float xx = fmaf(tt, edx, ex);
          xmn = fminf(xmn, xx);
          xmx = fmaxf(xmx, xx);
        }
      }
    }
  }
  s0 = 0;
  s1 = 0;
  if (xmx >= xmn) {
    s0 = max((int)floorf(xmn) - 1, 0);
    s1 = min((int)floorf(xmx) + 3, t.fw);
    if (s1 < s0) s1 = s0;
  }
}

// Per-unit setup of the raw-tap kernel (one thread per unit): the image's
// affine state (written by the image's first unit of this launch, read by
// the label kernel too) and the tile's footprint record.
__global__ void k_affine_setup_units(StepArgs a) {
  const int st = blockIdx.x * blockDim.x + threadIdx.x;
  if (st >= a.n_units * kAffSub) return;
  const int u = st / kAffSub, sub = st - u * kAffSub;
  const int2 unit = a.units[u];
  const int img = unit.x;
  const AfCoef cf = af_coef(a, img);
  ImgState s;
  for (int k = 0; k < 6; ++k) s.A[k] = cf.A[k];
  s.Af[0] = (float)cf.A[0]; s.Af[1] = (float)cf.A[1];
  s.Af[2] = (float)cf.A[3]; s.Af[3] = (float)cf.A[4];
  s.Wo = a.ddesc[img].width;
  s.Ho = a.ddesc[img].height;
  s.m = compose_exact(a.ops, a.tab, img, a.slot0 + 1, a.slot1, s.Wo, s.Ho);
  s.tiles_x = (s.Wo + kTileW - 1) / kTileW;
  s.pad = 0;
  if (sub == 0 && (u == 0 || a.units[u - 1].x != img))
    *reinterpret_cast<ImgState*>(reinterpret_cast<uint8_t*>(a.geo) + (size_t)img * kGeoBytes) = s;
  TileInfo t;
  const int tx0 = (unit.y & 0xffff) * kTileW, ty0 = (unit.y >> 16) * kTileH + sub * kRTH;
  const int tw = min(kTileW, s.Wo - tx0), th = max(min(kRTH, s.Ho - ty0), 0);
  if (th > 0) {
    tile_footprint(s, tx0, ty0, tw, th, t.fx0, t.fy0, t.fw, t.fh, t.vx, t.vy);
  } else {  // empty half of a short unit
    t.fx0 = t.fy0 = t.fw = t.fh = 0;
    for (int e = 0; e < 4; ++e) t.vx[e] = t.vy[e] = 0.f;
  }
  t.img = img;
  t.txy = tx0 | (ty0 << 16);
  t.twh = tw | (th << 16);
  const alb_image_desc sd = a.sdesc[img], dd = a.ddesc[img];
  for (int k = 0; k < 6; ++k) t.A[k] = s.A[k];
  for (int k = 0; k < 4; ++k) t.Af[k] = s.Af[k];
  t.m_ax = s.m.ax; t.m_bx = s.m.bx; t.m_ay = s.m.ay; t.m_by = s.m.by;
  t.Wo = s.Wo; t.Ho = s.Ho; t.Ws = sd.width; t.Hs = sd.height;
  t.soff = (long long)sd.offset; t.doff = (long long)dd.offset;
  t.spitch = sd.pitch; t.dpitch = dd.pitch;
  if (a.msdesc != nullptr && a.mddesc != nullptr) {
    const alb_image_desc msd = a.msdesc[img], mdd = a.mddesc[img];
    t.Wm = msd.width; t.Hm = msd.height; t.msoff = (long long)msd.offset; t.mdoff = (long long)mdd.offset;
    t.mspitch = msd.pitch; t.mdpitch = mdd.pitch;
  } else {
    t.Wm = t.Hm = 0; t.msoff = t.mdoff = 0; t.mspitch = t.mdpitch = 0;
  }
  // linear layout when no footprint row is reflected: row r of the footprint
  // at c0 + r * P with P = spitch (mod 16), so every row's 16-byte copies stay
  // aligned on both sides and a tap's shared address is affine in (x, y)
  t.P = 0;
  t.c0 = 0;
  if (th > 0 && t.fy0 >= 0 && t.fy0 + t.fh <= sd.height) {
    // P = spitch (mod 16), the smallest that holds a row; one more 16 bytes if
    // P / 4 is within 2 of a multiple of 32 words (every row in one bank: a
    // near-vertical walk of 32 lanes would hit one bank)
    const int base = 3 * t.fw + 46;
    int P = base + (((sd.pitch - base) % 16) + 16) % 16;
    const int wq = (P / 4) & 31;
    if (wq <= 2 || wq >= 30) P += 16;
    t.P = ((long long)t.fh * P + 32 <= kRRawBytes && fabs(s.A[3]) <= kRLinTan * fabs(s.A[0])) ? P : 0;
    const uintptr_t g0 = (uintptr_t)(a.src + sd.offset + (size_t)t.fy0 * sd.pitch) + (uintptr_t)(ptrdiff_t)(3 * t.fx0);
    t.c0 = 16 + (int)(g0 & 15);
  }
  for (int e = 0; e < 4; ++e) {
    const float dy = t.vy[(e + 1) & 3] - t.vy[e];
    t.eiy[e] = dy != 0.f ? 1.f / dy : 0.f;
  }
  for (int k = 0; k < 4; ++k) t.pad[k] = 0;
  const int xa = min(max(t.fx0, 0), sd.width), xb = max(min(t.fx0 + t.fw, sd.width), xa);
  const bool fill_rows = a.border != ALB_BORDER_REFLECT_101 && (t.fy0 < 0 || t.fy0 + t.fh > sd.height);
  const int ncols = fill_rows ? t.fw : (xa - t.fx0) + (t.fx0 + t.fw - xb);
  t.mb = magic_of((uint32_t)max(ncols, 1));
  reinterpret_cast<TileInfo*>(a.tiles)[st] = t;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(addr) : "memory");
  return v;
}

__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
  return v;
}

// issue the raw row copies of tile t: thread 2r + h copies chunks h, h + 2, ...
// of footprint row r into the rows at raw_a and writes rtab[2r + h] =
// rb[r + h] (shared address of the row's column fx0)
__device__ __forceinline__ void rt_stage(const StepArgs& a, const TileInfo& t, int* rtab, uint32_t raw_a,
                                         bool reflect, int tid) {
  const int fx0 = t.fx0, fy0 = t.fy0, fw = t.fw, fh = t.fh;
  if (!(fw <= kRMaxW && fh <= kRRows)) return;
  const int Ws = t.Ws, Hs = t.Hs;
  const uint8_t* simg = a.src + t.soff;
  const size_t spitch = (size_t)t.spitch;
  const int xa = min(max(fx0, 0), Ws), xb = max(min(fx0 + fw, Ws), xa);  // in-image columns [xa, xb)
  int* spans = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(rtab) + kROffSpan);
  for (int e = tid; e < kRTpr * fh; e += kRThreads) {
    const int r = e / kRTpr, h = e % kRTpr;
    int s0, s1;
    row_span(t, r, s0, s1);  // only the columns the rotated tile's taps reach
    if (h == 0) spans[r] = s0 | (s1 << 16);
    const int ca = max(xa, fx0 + s0), cb = min(xb, fx0 + s1);
    bool in;
    const int ry = border_idx(fy0 + r, Hs, reflect, in);
    const uintptr_t g = (uintptr_t)(simg + (size_t)(in ? ry : 0) * spitch) + (uintptr_t)(ptrdiff_t)(3 * fx0);
    // column fx0 of row r (address g) sits at B_r: c0 + r * P (linear layout) or
    // r * kRPitch + 16 + (g & 15) (row table); both keep B_r = g (mod 16)
    const int Br = t.P ? t.c0 + r * t.P : r * kRPitch + 16 + (int)(g & 15);
    if (in && cb > ca) {  // (no in-image column: the border pass fills the row)
      const uintptr_t g0 = g + 3 * (ca - fx0), ge = g0 + 3 * (cb - ca);
      const uint32_t d0 = raw_a + (uint32_t)Br - (uint32_t)g;
      for (uintptr_t gk = (g0 & ~(uintptr_t)15) + 16 * h; gk < ge; gk += 16 * kRTpr)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d0 + (uint32_t)gk), "l"(gk) : "memory");
    }
    // row-table entries rb[r] (h = 0) and rb[r + 1] (h = 1; the h = 0 thread too with one thread per row)
    for (int hh = h; hh < (kRTpr == 1 ? 2 : min(h + 1, 2)); ++hh) {
      const int rr = min(r + hh, fh - 1);
      int Brr = Br;
      if (hh) {
        bool in1;
        const int ry1 = border_idx(fy0 + rr, Hs, reflect, in1);
        const uintptr_t gr = (uintptr_t)(simg + (size_t)(in1 ? ry1 : 0) * spitch) + (uintptr_t)(ptrdiff_t)(3 * fx0);
        Brr = t.P ? t.c0 + rr * t.P : rr * kRPitch + 16 + (int)(gr & 15);
      }
      rtab[2 * r + hh] = (int)raw_a + Brr;
    }
  }
}

// border columns (x < 0 or x >= W) and constant-fill rows of a staged tile;
// returns whether it wrote anything (block-uniform)
__device__ __forceinline__ bool rt_border(const StepArgs& a, const TileInfo& t, const int* rtab, uint8_t* raw,
                                          uint32_t raw_a, bool reflect, int tid) {
  const int fx0 = t.fx0, fy0 = t.fy0, fw = t.fw, fh = t.fh;
  if (!(fw <= kRMaxW && fh <= kRRows)) return false;
  const int Ws = t.Ws, Hs = t.Hs;
  const uint8_t* simg = a.src + t.soff;
  const size_t spitch = (size_t)t.spitch;
  const int xa = min(max(fx0, 0), Ws), xb = max(min(fx0 + fw, Ws), xa);
  const int ncl = xa - fx0, nb = ncl + (fx0 + fw - xb);
  const bool fill_rows = !reflect && (fy0 < 0 || fy0 + fh > Hs);
  if (nb == 0 && !fill_rows) return false;
  const int ncols = fill_rows ? fw : nb;  // fill rows: every column
  const int* spans = reinterpret_cast<const int*>(reinterpret_cast<const uint8_t*>(rtab) + kROffSpan);
  for (int it = tid; it < fh * ncols; it += kRThreads) {
    const int r = fdiv(it, t.mb), j = it - r * ncols;
    const int sp = spans[r], s0 = sp & 0xffff, s1 = sp >> 16;
    bool rin;
    const int ry = border_idx(fy0 + r, Hs, reflect, rin);
    int c;
    if (fill_rows) {
      c = j;
      if (rin && c >= xa - fx0 && c < xb - fx0) continue;  // in-image pixel of a kept row
    } else {
      c = j < ncl ? j : (xb - fx0) + (j - ncl);
    }
    if (c < s0 || c >= s1) continue;  // no tap of the tile reads it
    const int rb = rtab[2 * r] - (int)raw_a;
    bool cin;
    const int rx = border_idx(fx0 + c, Ws, reflect, cin);
    uint32_t v;
    if (!rin || !cin) {
      v = a.fill;
    } else if (rx >= max(xa, fx0 + s0) && rx < min(xb, fx0 + s1)) {  // staged in this row
      const uint8_t* s = raw + rb + 3 * (rx - fx0);
      v = (uint32_t)s[0] | ((uint32_t)s[1] << 8) | ((uint32_t)s[2] << 16);
    } else {
      v = fetch_rgb(simg + (size_t)ry * spitch, rx);
    }
    uint8_t* d = raw + rb + 3 * c;
    d[0] = (uint8_t)v;
    d[1] = (uint8_t)(v >> 8);
    d[2] = (uint8_t)(v >> 16);
  }
  return true;
}

#ifndef ALB_RT_ROWUNROLL
#define ALB_RT_ROWUNROLL 1
#endif
constexpr int kRowUnroll = ALB_RT_ROWUNROLL;  // rows per unrolled step of the raw-tap kernel's row loop

template <int kOne, bool kMask>
#ifndef ALB_RT_MINB
#define ALB_RT_MINB (1024 / kRThreads)  // CTAs per SM (64-register cap)
#endif
__global__ void __launch_bounds__(kRThreads, ALB_RT_MINB) k_affine_rt(StepArgs a) {
  // kMask: the nearest label of every output pixel too (cfg3 / cfg5), from the
  // pixel's own coordinates -- the decision k_affine_mask makes -- gathered
  // straight from the source mask (L1-resident neighbourhood)
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  StageCtx x;
  init_stages(a, x);
  uint8_t* smb = reinterpret_cast<uint8_t*>(sm + x.n_lut * kLutWords);
  const bool reflect = a.border == ALB_BORDER_REFLECT_101;
  const TileInfo* tinfo = reinterpret_cast<const TileInfo*>(a.tiles);
  int* rtab = reinterpret_cast<int*>(smb + kROffTab);
  uint8_t* raw = smb + kROffRaw;
  const uint32_t tab_a = smem_u32(rtab), raw_a = smem_u32(raw);
  TileInfo* ctx = reinterpret_cast<TileInfo*>(smb + kRBuf);  // [2]: this tile's and the next tile's record
  // the record of tile v into ctx[k]: 16 threads x 16-byte cp.async
  auto prefetch = [&](int v, int k) {
    if (tid < kTileInfoBytes / 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(ctx + k) + 16u * tid),
                   "l"(reinterpret_cast<const uint8_t*>(tinfo + v) + 16 * tid)
                   : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  int u0, u1;
  unit_range(a.n_units, u0, u1);
  const int ubeg = u0 * kAffSub, uend = u1 * kAffSub;
  int lut_img = -1;
  if (ubeg < uend) prefetch(ubeg, 0);
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  for (int u = ubeg; u < uend; ++u) {
    const int cur = (u - ubeg) & 1;
    const TileInfo& t = ctx[cur];
    rt_stage(a, t, rtab, raw_a, reflect, tid);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const int img = t.img;
    const int fx0 = t.fx0, fy0 = t.fy0, fw = t.fw, fh = t.fh;
    const int tx0 = t.txy & 0xffff, ty0 = t.txy >> 16, tw = t.twh & 0xffff, th = t.twh >> 16;
    const bool fits = fw <= kRMaxW && fh <= kRRows;
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();  // tile u's rows landed
    bool bar = rt_border(a, t, rtab, raw, raw_a, reflect, tid);
    if (kOne != kStagesNone && img != lut_img) {  // LUTs are read only in the compute phase
      load_stages(a, img, sm, x, kRThreads);
      lut_img = img;
      bar = true;
    }
    if (bar) __syncthreads();
    if (u + 1 < uend) prefetch(u + 1, cur ^ 1);  // lands while this tile computes
    const int Ws = t.Ws, Hs = t.Hs;
    const uint8_t* simg = a.src + t.soff;
    const size_t spitch = (size_t)t.spitch;
    const int m_ax = t.m_ax, m_bx = t.m_bx, m_ay = t.m_ay, m_by = t.m_by;
    const int Wo = t.Wo;
    const float A0f = t.Af[0], A3f = t.Af[2];
    const size_t dpitch = (size_t)t.dpitch;
    uint8_t* drow0 = a.dst + t.doff + (size_t)ty0 * dpitch + (size_t)tx0 * 3;
    {
      const float2 A14 = make_float2(t.Af[1], t.Af[3]);
      int xw[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) xw[j] = m_ax * min(tx0 + lane + 32 * j, Wo - 1) + m_bx;
      const int row0 = warp * kRWarpRows;
      uint8_t* dlane = drow0 + 3 * lane;
      const int nrows = min(kRWarpRows, th - row0);
      // the body for one kind of tile (staged taps or global taps)
      // label gathers: the tile's nearest taps all inside the mask (footprint
      // test) -> no border resolution
      const uint8_t* msrc = nullptr;
      uint8_t* morow = nullptr;
      int mpitch = 0, Wm = 0, Hm = 0;
      size_t mdpitch = 0;
      bool minner = false;
      if constexpr (kMask) {
        msrc = a.msrc + t.msoff;
        mpitch = t.mspitch;
        Wm = t.Wm;
        Hm = t.Hm;
        mdpitch = (size_t)t.mdpitch;
        morow = a.mdst + t.mdoff + (size_t)(ty0 + row0) * mdpitch + tx0 + lane;
        minner = fx0 >= 0 && fy0 >= 0 && fx0 + fw <= Wm && fy0 + fh <= Hm;
      }
      const uint32_t lP = (uint32_t)t.P;
      auto rows = [&](auto staged, auto linear) {
        constexpr bool kStaged = decltype(staged)::value;
        constexpr bool kLinear = decltype(linear)::value;
        const bool st0 = lane < tw, st1 = lane + 32 < tw;
        const size_t pitch = dpitch;
        uint8_t* orow = dlane + (size_t)row0 * pitch;  // column lane; lane + 32 is 96 bytes on
        int i = 0;
        while (i < nrows) {  // segments of rows in one 16-row cell row (yw moves by m_ay = +-1)
          const int yw0 = m_ay * (ty0 + row0 + i) + m_by;
          const int cy = yw0 >> 4;
          const int iend = min(nrows, i + (m_ay > 0 ? 16 - (yw0 & 15) : (yw0 & 15) + 1));
          float2 bxy[2];
          uint32_t cxo[2], cyo[2];
          int aix[2], aiy[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {  // fp64 anchors of this cell row
            const Anchor an = cell_anchor(t.A, A0f, A3f, xw[j], cy);
            bxy[j] = make_float2(an.bx, an.by);
            aix[j] = an.ix;
            aiy[j] = an.iy;
            // tap byte address = rb[row] + 3 * qxb + cxo; row entry = 8 * qyb + cyo
            cxo[j] = 3u * (uint32_t)(an.ix - fx0) - 3u * kMagic15Bits;
            if constexpr (kLinear)  // tap address = P * qyb + 3 * qxb + cyo
              cyo[j] = raw_a + (uint32_t)t.c0 + lP * ((uint32_t)(an.iy - fy0) - kMagic15Bits) + cxo[j];
            else
              cyo[j] = tab_a + 8u * ((uint32_t)(an.iy - fy0) - kMagic15Bits);
          }
          float dyl = (float)(yw0 & 15);
          const float ddy = (float)m_ay;
#pragma unroll kRowUnroll
          for (; i < iend; ++i, dyl += ddy, orow += pitch) {
            uint32_t rr[2], gg[2], bb[2];
            [[maybe_unused]] uint8_t mv[2];  // labels (kMask)
#pragma unroll
            for (int j = 0; j < 2; ++j) {  // both columns always (clamped): the two pixels interleave
              const float2 l = __ffma2_rn(A14, make_float2(dyl, dyl), bxy[j]);
              const float2 tq = fadd2_rm(l, make_float2(kMagic15, kMagic15));  // floor + 1.5*2^23
              const float2 fl = __fadd2_rn(tq, make_float2(-kMagic15, -kMagic15));
              const float2 fr = __fadd2_rn(l, make_float2(-fl.x, -fl.y));
              const uint32_t qxb = __float_as_uint(tq.x), qyb = __float_as_uint(tq.y);
              if constexpr (kMask) {  // nearest: round half up
                const int nx = aix[j] + (int)(qxb - kMagic15Bits) + (fr.x >= 0.5f ? 1 : 0);
                const int ny = aiy[j] + (int)(qyb - kMagic15Bits) + (fr.y >= 0.5f ? 1 : 0);
                if (minner) {
                  mv[j] = __ldg(msrc + ny * mpitch + nx);
                } else {
                  bool ri, ci;
                  const int yy = border_idx(ny, Hm, reflect, ri), xx = border_idx(nx, Wm, reflect, ci);
                  mv[j] = (ri && ci) ? __ldg(msrc + yy * mpitch + xx) : (uint8_t)a.mask_fill;
                }
              }
              uint32_t r, g, b;
              if constexpr (kStaged) {
                uint32_t a0, a1;  // shared byte addresses of the two tap rows
                if constexpr (kLinear) {
                  a0 = qxb * 3u + (qyb * lP + cyo[j]);
                  a1 = a0 + lP;
                } else {
                  const uint32_t cb = qxb * 3u + cxo[j];
                  uint32_t ta;
                  asm("mad.lo.u32 %0, %1, 8, %2;" : "=r"(ta) : "r"(qyb), "r"(cyo[j]));
                  const uint2 rbp = lds64(ta);
                  a0 = rbp.x + cb;
                  a1 = rbp.y + cb;
                }
                const uint32_t b0 = a0 & ~3u, b1 = a1 & ~3u;
                const uint32_t w00 = lds32(b0), w01 = lds32(b0 + 4), w02 = lds32(b0 + 8);
                const uint32_t w10 = lds32(b1), w11 = lds32(b1 + 4), w12 = lds32(b1 + 8);
                const uint32_t s0 = a0 << 3, s1 = a1 << 3;
                bilerp3_raw(__funnelshift_r(w00, w01, s0), __funnelshift_r(w01, w02, s0),
                            __funnelshift_r(w10, w11, s1), __funnelshift_r(w11, w12, s1), fr, r, g, b);
              } else {  // footprint beyond the staging capacity: taps from global
                auto tap = [&](int px_, int py_) -> uint32_t {
                  bool ri, ci;
                  const int yy = border_idx(py_, Hs, reflect, ri), xx = border_idx(px_, Ws, reflect, ci);
                  return (ri && ci) ? fetch_rgb(simg + (size_t)yy * spitch, xx) : a.fill;
                };
                const int X = aix[j] + (int)(qxb - kMagic15Bits), Y = aiy[j] + (int)(qyb - kMagic15Bits);
                bilerp3(tap(X, Y), tap(X + 1, Y), tap(X, Y + 1), tap(X + 1, Y + 1), fr, r, g, b);
              }
              if constexpr (kOne != kStagesNone) {
                r &= 0xffu; g &= 0xffu; b &= 0xffu;
                apply_stages_t<kOne>(x, sm, lane, r, g, b);
              }
              rr[j] = r; gg[j] = g; bb[j] = b;
            }
            // straight to global: a warp's byte stores cover 96 contiguous bytes
            if (st0) { orow[0] = (uint8_t)rr[0]; orow[1] = (uint8_t)gg[0]; orow[2] = (uint8_t)bb[0]; }
            if (st1) { orow[96] = (uint8_t)rr[1]; orow[97] = (uint8_t)gg[1]; orow[98] = (uint8_t)bb[1]; }
            if constexpr (kMask) {
              if (st0) morow[0] = mv[0];
              if (st1) morow[32] = mv[1];
              morow += mdpitch;
            }
          }
        }
      };
      if (fits && lP != 0) rows(std::true_type{}, std::true_type{});
      else if (fits) rows(std::true_type{}, std::false_type{});
      else rows(std::false_type{}, std::false_type{});
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");  // the next tile's record landed
    __syncthreads();  // tile consumed: raw rows free
  }
}

// Nearest-label mask warp beside the pipelined image kernel (cfg3 / cfg5):
// the same fp64 cell anchors and fp32 local offsets as the image kernels, so
// a mask pixel takes the label at its image source coordinate rounded half up
// -- exactly the decision the fused masked kernel makes.  One
// CTA per 64 x 64 output tile; labels are read straight from global (1 byte
// per pixel, L1/L2 resident neighbourhood).
// kFast: a full 64 x 64 tile whose nearest taps all lie inside the source
// mask (decided per tile from its fp64 corner coordinates, with a 1-pixel
// margin): no border resolution, no row / column predicates.
template <bool kFast>
__device__ __forceinline__ void affine_mask_tile(const StepArgs& a, const ImgState& is, int img, int tx0, int ty0,
                                                 int tw, int th) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const alb_image_desc msd = a.msdesc[img], mdd = a.mddesc[img];
  const uint8_t* msrc = a.msrc + msd.offset;
  uint8_t* mdst = a.mdst + mdd.offset + (size_t)ty0 * mdd.pitch + tx0;
  const bool reflect = a.border == ALB_BORDER_REFLECT_101;
  const float2 A14 = make_float2(is.Af[1], is.Af[3]);
  const int ncol = kFast ? 2 : (tw > 32 ? 2 : 1);
  int xw[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) xw[j] = is.m.ax * min(tx0 + lane + 32 * j, is.Wo - 1) + is.m.bx;
  // warp w owns the contiguous rows [8w, 8w + 8): at most two cell rows of
  // fp64 anchors; all 16 label addresses first, then 16 independent loads
  constexpr int kR = kTileH / (kAfThreads / 32);
  int cur_cy = -0x7fffffff;
  float2 bxy[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  int aix[2] = {0, 0}, aiy[2] = {0, 0};
  int src_off[kR][2];  // label offset in the source mask, or -1 for the fill
#pragma unroll
  for (int i = 0; i < kR; ++i) {
    const int row = warp * kR + i;
    src_off[i][0] = src_off[i][1] = -1;
    if (!kFast && row >= th) continue;
    const int yw = is.m.ay * (ty0 + row) + is.m.by;
    if ((yw >> 4) != cur_cy) {
      cur_cy = yw >> 4;
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (j < ncol) {
          const Anchor an = cell_anchor(is.A, is.Af[0], is.Af[2], xw[j], cur_cy);
          bxy[j] = make_float2(an.bx, an.by);
          aix[j] = an.ix;
          aiy[j] = an.iy;
        }
      }
    }
    const float dyl = (float)(yw & 15);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float2 l = __ffma2_rn(A14, make_float2(dyl, dyl), bxy[j]);
      const float2 tq = fadd2_rm(l, make_float2(kMagic15, kMagic15));
      const float2 fl = __fadd2_rn(tq, make_float2(-kMagic15, -kMagic15));
      const float2 fr = __fadd2_rn(l, make_float2(-fl.x, -fl.y));
      const int nx = aix[j] + (int)(__float_as_uint(tq.x) - kMagic15Bits) + (fr.x >= 0.5f ? 1 : 0);
      const int ny = aiy[j] + (int)(__float_as_uint(tq.y) - kMagic15Bits) + (fr.y >= 0.5f ? 1 : 0);
      if constexpr (kFast) {
        src_off[i][j] = ny * msd.pitch + nx;
      } else {
        bool ri, ci;
        const int yy = border_idx(ny, msd.height, reflect, ri);
        const int xx = border_idx(nx, msd.width, reflect, ci);
        src_off[i][j] = (ri && ci) ? yy * msd.pitch + xx : -1;
      }
    }
  }
  uint8_t v[kR][2];
#pragma unroll
  for (int i = 0; i < kR; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      v[i][j] = (kFast || src_off[i][j] >= 0) ? __ldg(msrc + src_off[i][j]) : (uint8_t)a.mask_fill;
#pragma unroll
  for (int i = 0; i < kR; ++i) {
    const int row = warp * kR + i;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c = lane + 32 * j;
      if (kFast || (row < th && j < ncol && c < tw)) mdst[(size_t)row * mdd.pitch + c] = v[i][j];
    }
  }
}

__global__ void __launch_bounds__(kAfThreads, 4) k_affine_mask(StepArgs a) {
  const int2 unit = a.units[blockIdx.x];
  const int img = unit.x;
  __shared__ ImgState sis;  // per-image state, one word per thread
  __shared__ int s_fast;
  const int tx0 = (unit.y & 0xffff) * kTileW, ty0 = (unit.y >> 16) * kTileH;
  {
    constexpr int kW = (int)sizeof(ImgState) / 4;
    const uint32_t* gsrc = reinterpret_cast<const uint32_t*>(reinterpret_cast<const uint8_t*>(a.geo) +
                                                             (size_t)img * kGeoBytes);
    if (threadIdx.x < kW) reinterpret_cast<uint32_t*>(&sis)[threadIdx.x] = __ldcg(gsrc + threadIdx.x);
    if (threadIdx.x == 32) {  // interior test from the tile's fp64 corners (1 px margin)
      const ImgState& g = *reinterpret_cast<const ImgState*>(gsrc);
      const int Wo = __ldcg(&g.Wo), Ho = __ldcg(&g.Ho);
      const int tw = min(kTileW, Wo - tx0), th = min(kTileH, Ho - ty0);
      int fast = tw == kTileW && th == kTileH;
      if (fast) {
        const int ax = __ldcg(&g.m.ax), bx = __ldcg(&g.m.bx), ay = __ldcg(&g.m.ay), by = __ldcg(&g.m.by);
        double A[6];
        for (int q = 0; q < 6; ++q) A[q] = __ldcg(&g.A[q]);
        const double xa = ax * tx0 + bx, xb = ax * (tx0 + tw - 1) + bx;
        const double ya = ay * ty0 + by, yb = ay * (ty0 + th - 1) + by;
        double lx = 1e300, hx = -1e300, ly = 1e300, hy = -1e300;
        for (int c = 0; c < 4; ++c) {
          const double xw = (c & 1) ? xb : xa, yw = (c & 2) ? yb : ya;
          const double sx = fma(A[0], xw, fma(A[1], yw, A[2])), sy = fma(A[3], xw, fma(A[4], yw, A[5]));
          lx = fmin(lx, sx); hx = fmax(hx, sx); ly = fmin(ly, sy); hy = fmax(hy, sy);
        }
        const alb_image_desc msd = a.msdesc[img];
        fast = floor(lx) - 1.0 >= 0.0 && floor(hx) + 2.0 <= (double)(msd.width - 1) && floor(ly) - 1.0 >= 0.0 &&
               floor(hy) + 2.0 <= (double)(msd.height - 1);
      }
      s_fast = fast;
    }
    __syncthreads();
  }
  const ImgState& is = sis;
  const int tw = min(kTileW, is.Wo - tx0), th = min(kTileH, is.Ho - ty0);
  if (s_fast) affine_mask_tile<true>(a, is, img, tx0, ty0, tw, th);
  else affine_mask_tile<false>(a, is, img, tx0, ty0, tw, th);
}

static size_t affine_smem(const StepArgs& a) {
  return (size_t)count_lut_stages(a) * kLutWords * 4 + kOffStage + (size_t)a.unit_size * 4 + 16 +
         (a.mdst ? (size_t)(kTileH * kMobPitch + kMStageBytes) : 0);
}

template <int kOne, bool kMask, int kMode>
static void launch_affine_v(const StepArgs& a, size_t smem, cudaStream_t s) {
  persistent_grid((const void*)k_affine<kOne, kMask, kMode>, kAfThreads, smem, a.n_units);  // smem attribute
  k_affine<kOne, kMask, kMode><<<a.n_units, kAfThreads, smem, s>>>(a);  // one CTA per tile
}

// the raw-tap kernel serves the bilinear u8 path (ALB_AFFINE_PIPE=1 selects
// the pipelined kernel instead, an A/B switch kept for measurements)
static bool affine_fast(const StepArgs& a) {
  return !(a.interp == ALB_INTERP_NEAREST || a.normalize || a.min_scale < 0.9f || a.unit_size < 14040);
}

static bool affine_rt(const StepArgs& a) { return affine_fast(a) && std::getenv("ALB_AFFINE_PIPE") == nullptr; }

template <int kOne>
static void launch_affine_t(const StepArgs& a, size_t smem, cudaStream_t s) {
  // fast variant always stages: a 64x64 tile's footprint (+halo) at scale
  // >= 0.9 is at most fw, fh <= 104 and S <= fw + 31, i.e. <= 14040 words
  const bool generic = !affine_fast(a);
  const bool mask = a.mdst != nullptr;
  if (generic) {
    if (mask) launch_affine_v<kOne, true, 1>(a, smem, s);
    else launch_affine_v<kOne, false, 1>(a, smem, s);
  } else {  // pipelined TMA-staged path; masks (cfg3 / cfg5) through the label kernel beside it
    StepArgs ai = a;
    ai.msrc = nullptr;
    ai.mdst = nullptr;
    const size_t psmem = (size_t)count_lut_stages(a) * kLutWords * 4 + kPSmem;
    // ~16 tiles per CTA: long enough to pipeline, short enough that the
    // hardware re-balances CTAs across SMs (measured: 16 > 8, 32 > persistent)
    const int grid = std::max(persistent_grid((const void*)k_affine_pipe<kOne>, kPThreads, psmem, a.n_units),
                              (a.n_units + 15) / 16);
    if (!affine_rt(a)) {  // A/B switch: the round-2 pipelined kernel; labels beside it
      if (mask) k_affine_mask<<<a.n_units, kAfThreads, 0, side_fork(s)>>>(a);  // side stream (fork / join)
      k_affine_pipe<kOne><<<grid, kPThreads, psmem, s>>>(ai);
      if (mask) side_join(s);
    } else {
      const size_t rsmem = (size_t)count_lut_stages(a) * kLutWords * 4 + kRSmem;
#ifndef ALB_RT_TPC
#define ALB_RT_TPC 8  // units per CTA (0: one persistent wave, units split evenly; measured 8 < 16 < 32 < 0)
#endif
      const void* fn = mask ? (const void*)k_affine_rt<kOne, true> : (const void*)k_affine_rt<kOne, false>;
      const int pg = persistent_grid(fn, kRThreads, rsmem, a.n_units);
      const int rgrid = ALB_RT_TPC > 0 ? std::max(pg, (a.n_units + ALB_RT_TPC - 1) / ALB_RT_TPC) : pg;
      if (mask) k_affine_rt<kOne, true><<<rgrid, kRThreads, rsmem, s>>>(a);  // image + labels in one kernel
      else k_affine_rt<kOne, false><<<rgrid, kRThreads, rsmem, s>>>(ai);
    }
  }
}

void launch_affine(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  if (affine_rt(a))  // per-image state + per-tile footprints
    k_affine_setup_units<<<(a.n_units * kAffSub + 127) / 128, 128, 0, s>>>(a);
  else  // per-image state for both kernels
    k_affine_setup<<<(a.n_img - a.img0 + 127) / 128, 128, 0, s>>>(a);
  const size_t smem = affine_smem(a);
  const int mode = stage_mode(a);
  ALB_DISPATCH_STAGES(mode, launch_affine_t, a, smem, s)
}

}  // namespace alb
