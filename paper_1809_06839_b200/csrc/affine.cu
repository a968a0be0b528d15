// affine.cu -- K4 Rotate / ShiftScaleRotate (O7) with fused post
// ops (K10: RandomCrop / Crop / flips on the output coordinates), the
// pointwise stage chain, Normalize output and the nearest-neighbour mask.
//
// Inverse map per warp-output pixel (xw, yw):
//   x_s = cx + (cos*(xw-cx-tx) - sin*(yw-cy-ty)) / s,  likewise y_s,
// written as x_s = A0*xw + A1*yw + A2 with the coefficients formed in fp64.
// Coordinates: an fp64 ANCHOR per 16x16 cell of warp-output coordinates
// (split into integer + fp32 fraction) plus fp32 local offsets (<= 15 px):
// error ~2e-6 px, and a pixel's value depends only on its warp-output
// coordinates, so the fused cfg5 kernel equals the unfused kernel bit for bit.
//
// Work unit = (image, 64x32 output tile); persistent grid over contiguous
// unit ranges.  Per tile:
//  1. thread 0 derives the source footprint, the bank-friendly staged stride
//     S (= +-1 mod 32 from the rotation, so 32 consecutive output pixels hit
//     distinct banks) and every division constant of the tile;
//  2. the footprint (+ bilinear halo) is staged in shared memory as RGBx
//     words with the border resolved per staged pixel (reflect-101 or
//     constant): interior runs of 16 pixels with 16-byte loads (two runs in
//     flight per thread), border pixels one per thread;
//  3. each warp owns 4 output rows, lane = column, 2 pixels per lane per row:
//     anchored coordinates, magic-number floor, 4 shared taps, paired-fp32
//     blend, one RGBx word into the shared output tile;
//  4. the tile is repacked RGBx -> RGB in shared memory and written with
//     aligned 16-byte stores.
// Footprints larger than the staging capacity fall back to per-tap loads.
#include <algorithm>

#include "stages.cuh"

namespace alb {

constexpr int kAfThreads = 256;
constexpr int kAfWarps = kAfThreads / 32;
constexpr int kTileW = 64, kTileH = 64;
constexpr int kRowsPerWarp = kTileH / kAfWarps;
constexpr int kTilePitch = kTileW * 3 + 16;  // packed RGB tile row pitch (bytes, 16-aligned)

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

__device__ __forceinline__ uint32_t fetch_rgb(const uint8_t* row, int x) {
  const uint8_t* p = row + 3 * x;
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16);
}

// border index: one reflection without modulo (the common case), else general
__device__ __forceinline__ int border_idx(int i, int n, bool reflect, bool& in) {
  if (i >= 0 && i < n) { in = true; return i; }
  if (!reflect) { in = false; return 0; }
  in = true;
  int k = i < 0 ? -i : i;
  if (k >= n) k = 2 * n - 2 - k;
  return (k >= 0 && k < n) ? k : reflect101(i, n);
}

// floor(v) for |v| < 2^22 via round-down add of 1.5*2^23: returns the
// integer and the exact fraction v - floor(v)
__device__ __forceinline__ int floor_frac(float v, float& frac) {
  const float M = 12582912.f;  // 1.5 * 2^23
  const float t = __fadd_rd(v, M);
  frac = v - (t - M);
  return __float_as_int(t) - 0x4B400000;
}

struct TileGeom {
  int fx0, fy0, S, fw, fh, staged, Sm, ci0, ci1, nvi, P, tail;
  uint32_t m_nvi, m_P, m_fw, m_copy;
};

struct ImgState {
  double A[6];
  float Af[4];
  Map1 m;
  int Wo, Ho, tiles_x, pad;
};

// smem word offsets (from sm + n_lut * kLutWords)
constexpr int kOffIs = 0;
constexpr int kOffTg = (int)(sizeof(ImgState) + 15) / 16 * 4;
constexpr int kOffTile = kOffTg + (int)(sizeof(TileGeom) + 15) / 16 * 4;          // RGBx [32][64]
constexpr int kOffStage = kOffTile + kTileH * kTileW;
// the packed RGB output tile [64][208] aliases the stage buffer: it is written
// only after the compute pass has consumed the staged footprint
static_assert(kTileH * kTilePitch + 16 <= 14040 * 4, "pack must fit in the stage buffer");

// kGeneric = false: bilinear, no mask, u8 output (the single-op and cfg5-image
// fast path) -- the uniform mode branches compile away.
template <int kOne, bool kGeneric>
__global__ void __launch_bounds__(kAfThreads, 3) k_affine(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  StageCtx x;
  init_stages(a, x);
  const int base = x.n_lut * kLutWords;
  ImgState* is = reinterpret_cast<ImgState*>(sm + base + kOffIs);
  TileGeom* tg = reinterpret_cast<TileGeom*>(sm + base + kOffTg);
  uint32_t* tile = sm + base + kOffTile;
  uint32_t* stage = sm + base + kOffStage;
  uint8_t* pack = reinterpret_cast<uint8_t*>(stage);  // aliases stage (see kOffStage)
  uint8_t* mstage = reinterpret_cast<uint8_t*>(stage + a.unit_size);
  const bool reflect = a.border == ALB_BORDER_REFLECT_101;
  const bool nearest = kGeneric && a.interp == ALB_INTERP_NEAREST;
  const bool has_mask = kGeneric && a.mdst != nullptr;
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
      if (threadIdx.x == 0) {
        const AfCoef cf = af_coef(a, img);
        ImgState s;
        for (int k = 0; k < 6; ++k) s.A[k] = cf.A[k];
        s.Af[0] = (float)cf.A[0]; s.Af[1] = (float)cf.A[1];
        s.Af[2] = (float)cf.A[3]; s.Af[3] = (float)cf.A[4];
        s.Wo = a.normalize ? a.out_w : a.ddesc[img].width;
        s.Ho = a.normalize ? a.out_h : a.ddesc[img].height;
        s.m = compose_exact(a.ops, a.tab, img, a.slot0 + 1, a.slot1, s.Wo, s.Ho);
        s.tiles_x = (s.Wo + kTileW - 1) / kTileW;
        *is = s;
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
    if (warp == 0) {  // tile geometry: corners on lanes 0-3, division constants on lanes 0-3
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
      TileGeom t;
      t.fx0 = (int)floor(lx) - 1;
      t.fy0 = (int)floor(ly) - 1;
      t.fw = (int)floor(hx) + 2 - t.fx0 + 1;
      t.fh = (int)floor(hy) + 2 - t.fy0 + 1;
      const int want = fabs(A[0] + A[3]) >= fabs(A[0] - A[3]) ? 1 : 31;  // lane step +-(A0 + S*A3)
      t.S = t.fw + ((want - t.fw % 32) + 32) % 32;
      t.Sm = (t.fw + 3) & ~3;
      t.staged = (long long)t.S * t.fh <= a.unit_size &&
                 (!has_mask || (long long)t.Sm * t.fh <= a.unit_size);
      t.ci0 = min(max(-t.fx0, 0), t.fw);
      t.ci1 = min(max(Ws - t.fx0, 0), t.fw);
      t.nvi = (t.ci1 - t.ci0 + 15) >> 4;  // last run of a row may be partial
      t.tail = 0;
      t.P = t.ci0 + (t.fw - t.ci1);        // border columns only
      // one integer division per lane instead of four in a row
      const uint32_t dv = lane == 0 ? (uint32_t)t.nvi : lane == 1 ? (uint32_t)t.P
                        : lane == 2 ? (uint32_t)t.fw : (uint32_t)((3 * tw) >> 4) + 2u;
      const uint32_t mg = magic_of(dv);
      t.m_nvi = __shfl_sync(0xffffffffu, mg, 0);
      t.m_P = __shfl_sync(0xffffffffu, mg, 1);
      t.m_fw = __shfl_sync(0xffffffffu, mg, 2);
      t.m_copy = __shfl_sync(0xffffffffu, mg, 3);
      if (lane == 0) *tg = t;
    }
    __syncthreads();
    const TileGeom t = *tg;
    const uint8_t* simg = a.src + sd.offset;
    if (t.staged) {
      // pass A: 16-pixel interior runs with 16-byte loads, two runs in flight
      const int na = t.fh * t.nvi;
      for (int it = threadIdx.x; it < na; it += 2 * kAfThreads) {
        uint32_t w[2][12];
        int dst[2], nw[2];
        bool live[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int ik = it + k * kAfThreads;
          live[k] = ik < na;
          dst[k] = -1;
          nw[k] = 0;
          if (live[k]) {
            const int r = fdiv(ik, t.m_nvi);
            const int c = t.ci0 + ((ik - r * t.nvi) << 4);
            nw[k] = min(16, t.ci1 - c);  // partial last run of the row
            bool row_in;
            const int ry = border_idx(t.fy0 + r, Hs, reflect, row_in);
            dst[k] = r * t.S + c;
            if (row_in) {
              const uint8_t* srow = simg + (size_t)ry * sd.pitch;
              load_window<12>(srow + (size_t)(t.fx0 + c) * 3, srow, srow + (size_t)Ws * 3, w[k]);
            } else {
              live[k] = false;  // constant-border row
              for (int i = 0; i < nw[k]; ++i) stage[dst[k] + i] = a.fill;
            }
          }
        }
#pragma unroll
        for (int k = 0; k < 2; ++k)
          if (live[k]) {
            if (nw[k] == 16) {
#pragma unroll
              for (int i = 0; i < 16; ++i) stage[dst[k] + i] = rgbx_of(w[k], i);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                if (i < nw[k]) stage[dst[k] + i] = rgbx_of(w[k], i);
            }
          }
      }
      // pass B: border columns, one pixel per thread
      for (int it = threadIdx.x; it < t.fh * t.P; it += kAfThreads) {
        const int r = fdiv(it, t.m_P);
        const int j = it - r * t.P;
        const int c = j < t.ci0 ? j : t.ci1 + (j - t.ci0);
        bool row_in, col_in;
        const int ry = border_idx(t.fy0 + r, Hs, reflect, row_in);
        const int rx = border_idx(t.fx0 + c, Ws, reflect, col_in);
        stage[r * t.S + c] = (row_in && col_in) ? fetch_rgb(simg + (size_t)ry * sd.pitch, rx) : a.fill;
      }
      if (has_mask) {
        const uint8_t* smk = a.msrc + a.msdesc[img].offset;
        const int mpitch = a.msdesc[img].pitch;
        for (int it = threadIdx.x; it < t.fh * t.fw; it += kAfThreads) {
          const int r = fdiv(it, t.m_fw);
          const int c = it - r * t.fw;
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
    int xw[2];
    float dxl[2];
    int cur_cy[2] = {-0x7fffffff, -0x7fffffff};
    int abase[2] = {0, 0}, aix[2] = {0, 0}, aiy[2] = {0, 0};
    float afx[2] = {0.f, 0.f}, afy[2] = {0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      xw[j] = m.ax * min(tx0 + lane + 32 * j, Wo - 1) + m.bx;
      dxl[j] = (float)(xw[j] & 15);
    }
    if constexpr (!kGeneric) {
      // fast path (always staged, bilinear, u8 out): the lane's two pixels are
      // independent chains interleaved for ILP; columns >= tw compute clamped
      // garbage that the copy-out never reads.
      for (int i = 0; i < kRowsPerWarp; ++i) {
        const int row = warp * kRowsPerWarp + i;
        if (row >= th) break;
        const int yw = m.ay * (ty0 + row) + m.by;
        const float dyl = (float)(yw & 15);
        if ((yw >> 4) != cur_cy[0]) {  // warp-uniform: both columns share the cell row
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            cur_cy[j] = yw >> 4;
            const double xa = (double)((xw[j] >> 4) * 16), ya = (double)(cur_cy[j] * 16);
            const double sx = fma(A[0], xa, fma(A[1], ya, A[2]));
            const double sy = fma(A[3], xa, fma(A[4], ya, A[5]));
            const double flx = floor(sx), fly = floor(sy);
            afx[j] = (float)(sx - flx); afy[j] = (float)(sy - fly);
            abase[j] = ((int)fly - t.fy0) * t.S + ((int)flx - t.fx0);
          }
        }
        float fx[2], fy[2];
        int idx[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const float lx = fmaf(A0f, dxl[j], fmaf(A1f, dyl, afx[j]));
          const float ly = fmaf(A3f, dxl[j], fmaf(A4f, dyl, afy[j]));
          const int qx = floor_frac(lx, fx[j]), qy = floor_frac(ly, fy[j]);
          idx[j] = abase[j] + qy * t.S + qx;
        }
        uint32_t tp[2][4];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          tp[j][0] = stage[idx[j]];
          tp[j][1] = stage[idx[j] + 1];
          tp[j][2] = stage[idx[j] + t.S];
          tp[j][3] = stage[idx[j] + t.S + 1];
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint32_t px = bilerp_rgbx(tp[j][0], tp[j][1], tp[j][2], tp[j][3], fx[j], fy[j]);
          if (kOne != kStagesNone) {
            uint32_t r = px & 0xff, g = (px >> 8) & 0xff, b = (px >> 16) & 0xff;
            apply_stages_t<kOne>(x, sm, lane, r, g, b);
            px = r | (g << 8) | (b << 16);
          }
          tile[row * kTileW + lane + 32 * j] = px;
        }
      }
    } else
    for (int i = 0; i < kRowsPerWarp; ++i) {
      const int row = warp * kRowsPerWarp + i;
      if (row >= th) break;
      const int yo = ty0 + row;
      const int yw = m.ay * yo + m.by;
      const float dyl = (float)(yw & 15);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = lane + 32 * j;
        if (j == 1 && tw <= 32) break;
        if ((yw >> 4) != cur_cy[j]) {  // fp64 anchor of this column's 16x16 cell
          cur_cy[j] = yw >> 4;
          const double xa = (double)((xw[j] >> 4) * 16), ya = (double)(cur_cy[j] * 16);
          const double sx = fma(A[0], xa, fma(A[1], ya, A[2]));
          const double sy = fma(A[3], xa, fma(A[4], ya, A[5]));
          const double flx = floor(sx), fly = floor(sy);
          aix[j] = (int)flx; aiy[j] = (int)fly;
          afx[j] = (float)(sx - flx); afy[j] = (float)(sy - fly);
          abase[j] = (aiy[j] - t.fy0) * t.S + (aix[j] - t.fx0);
        }
        const float lx = fmaf(A0f, dxl[j], fmaf(A1f, dyl, afx[j]));
        const float ly = fmaf(A3f, dxl[j], fmaf(A4f, dyl, afy[j]));
        uint32_t px;
        if (nearest) {
          float f0, f1;
          const int qx = floor_frac(lx + 0.5f, f0), qy = floor_frac(ly + 0.5f, f1);
          if (t.staged) {
            px = stage[abase[j] + qy * t.S + qx];
          } else {
            bool ri, ci;
            const int yy = border_idx(aiy[j] + qy, Hs, reflect, ri);
            const int xx = border_idx(aix[j] + qx, Ws, reflect, ci);
            px = (ri && ci) ? fetch_rgb(simg + (size_t)yy * sd.pitch, xx) : a.fill;
          }
        } else {
          float fx, fy;
          const int qx = floor_frac(lx, fx), qy = floor_frac(ly, fy);
          uint32_t t00, t10, t01, t11;
          if (!kGeneric || t.staged) {
            const int idx = abase[j] + qy * t.S + qx;
            t00 = stage[idx]; t10 = stage[idx + 1]; t01 = stage[idx + t.S]; t11 = stage[idx + t.S + 1];
          } else {
            auto tap = [&](int px_, int py_) -> uint32_t {
              bool ri, ci;
              const int yy = border_idx(py_, Hs, reflect, ri), xx = border_idx(px_, Ws, reflect, ci);
              return (ri && ci) ? fetch_rgb(simg + (size_t)yy * sd.pitch, xx) : a.fill;
            };
            const int X = aix[j] + qx, Y = aiy[j] + qy;
            t00 = tap(X, Y); t10 = tap(X + 1, Y); t01 = tap(X, Y + 1); t11 = tap(X + 1, Y + 1);
          }
          px = bilerp_rgbx(t00, t10, t01, t11, fx, fy);
        }
        if (kOne != kStagesNone) {
          uint32_t r = px & 0xff, g = (px >> 8) & 0xff, b = (px >> 16) & 0xff;
          apply_stages_t<kOne>(x, sm, lane, r, g, b);
          px = r | (g << 8) | (b << 16);
        }
        if (normalize) {
          const size_t plane = (size_t)Ho * Wo;
          float* o = a.nchw + (size_t)img * 3 * plane + (size_t)yo * Wo + tx0 + c;
          const float* nl = a.tab.norm_lut;
          __stcs(o, nl[px & 0xff]);
          __stcs(o + plane, nl[256 + ((px >> 8) & 0xff)]);
          __stcs(o + 2 * plane, nl[512 + ((px >> 16) & 0xff)]);
        } else {
          tile[row * kTileW + c] = px;
        }
        if (has_mask) {
          float f0, f1;
          const int qx = floor_frac(lx + 0.5f, f0), qy = floor_frac(ly + 0.5f, f1);
          uint8_t v;
          if (t.staged) {
            v = mstage[(aiy[j] + qy - t.fy0) * t.Sm + (aix[j] + qx - t.fx0)];
          } else {
            bool ri, ci;
            const int yy = border_idx(aiy[j] + qy, Hs, reflect, ri);
            const int xx = border_idx(aix[j] + qx, Ws, reflect, ci);
            v = (ri && ci) ? a.msrc[a.msdesc[img].offset + (size_t)yy * a.msdesc[img].pitch + xx]
                           : (uint8_t)a.mask_fill;
          }
          if (c < tw) {
            const alb_image_desc mdd = a.mddesc[img];
            a.mdst[mdd.offset + (size_t)yo * mdd.pitch + tx0 + c] = v;
          }
        }
      }
    }
    if (!normalize) {
      __syncthreads();
      // repack RGBx -> RGB: 4 pixels (one 16-byte read) -> 12 bytes per thread item
      for (int it = threadIdx.x; it < kTileH * (kTileW / 4); it += kAfThreads) {
        const int r = it >> 4, q = it & 15;
        const uint4 v = *reinterpret_cast<const uint4*>(tile + r * kTileW + 4 * q);
        uint32_t* d = reinterpret_cast<uint32_t*>(pack + r * kTilePitch + 12 * q);
        d[0] = __byte_perm(v.x, v.y, 0x4210);
        d[1] = __byte_perm(v.y, v.z, 0x5421);
        d[2] = __byte_perm(v.z, v.w, 0x6542);
      }
      __syncthreads();
      const alb_image_desc dd = a.ddesc[img];
      cta_copy_rows(a.dst + dd.offset + (size_t)ty0 * dd.pitch + (size_t)tx0 * 3, dd.pitch, pack,
                    kTilePitch, th, 3 * tw, kAfThreads, t.m_copy);
    }
  }
}

static size_t affine_smem(const StepArgs& a) {
  return ((size_t)count_lut_stages(a) * kLutWords + kOffStage) * 4 + (size_t)a.unit_size * 4 +
         (a.mdst ? (size_t)a.unit_size : 0);
}

template <int kOne, bool kGeneric>
static void launch_affine_v(const StepArgs& a, size_t smem, cudaStream_t s) {
  const int grid = persistent_grid((const void*)k_affine<kOne, kGeneric>, kAfThreads, smem, a.n_units);
  k_affine<kOne, kGeneric><<<grid, kAfThreads, smem, s>>>(a);
}

template <int kOne>
static void launch_affine_t(const StepArgs& a, size_t smem, cudaStream_t s) {
  // fast variant always stages: a 64x64 tile's footprint (+halo) is at most
  // (63*sqrt2/s + 5 + 31) x (63*sqrt2/s + 5) words, <= 14040 <= a.unit_size for s >= 0.9
  const bool generic = a.interp == ALB_INTERP_NEAREST || a.mdst != nullptr || a.normalize ||
                       a.min_scale < 0.9f || a.unit_size < 14040;
  if (generic) launch_affine_v<kOne, true>(a, smem, s);
  else launch_affine_v<kOne, false>(a, smem, s);
}

void launch_affine(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  const size_t smem = affine_smem(a);
  const int mode = stage_mode(a);
  ALB_DISPATCH_STAGES(mode, launch_affine_t, a, smem, s)
}

}  // namespace alb
