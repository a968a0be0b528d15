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
// Work unit = (image, 64x32 output tile); the grid is persistent over
// contiguous unit ranges.  Per tile the source footprint (+ bilinear halo) is
// staged in shared memory as RGBx words with the border resolved per staged
// pixel (reflect-101 or constant fill): interior runs of 16 pixels with
// 16-byte loads, border pixels one per thread, so the hot loop has no border
// logic.  The staged row stride S is = +-1 (mod 32), picked from the rotation
// so 32 consecutive output pixels hit distinct banks.  Each warp owns 4 output
// rows (lane = column, 2 pixels per lane per row); RGB bytes go to a per-warp
// row buffer that the warp writes out with aligned 16-byte stores.
// Footprints larger than the staging capacity fall back to per-tap loads.
#include <algorithm>

#include "stages.cuh"

namespace alb {

constexpr int kAfThreads = 256;
constexpr int kAfWarps = kAfThreads / 32;
constexpr int kTileW = 64, kTileH = 32;
constexpr int kRowsPerWarp = kTileH / kAfWarps;
constexpr int kTilePitch = kTileW * 3 + 16;  // output tile row pitch in shared memory (16-aligned)

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

struct TileGeom {
  int fx0, fy0, S, fw, fh, staged, Sm, ci0, ci1, pad[3];
};

struct ImgState {
  double A[6];
  float Af[4];
  Map1 m;
  int Wo, Ho, tiles_x, pad;
};

// kGeneric = false: bilinear, no mask, u8 output (the single-op and cfg5-image
// fast path) -- the uniform mode branches compile away.
template <int kOne, bool kGeneric>
__global__ void __launch_bounds__(kAfThreads, 3) k_affine(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  StageCtx x;
  init_stages(a, x);
  ImgState* is = reinterpret_cast<ImgState*>(sm + x.n_lut * kLutWords);
  TileGeom* tg = reinterpret_cast<TileGeom*>(is + 1);
  uint8_t* tilebuf = reinterpret_cast<uint8_t*>(tg + 1);  // output tile, RGB bytes
  uint32_t* stage = reinterpret_cast<uint32_t*>(tilebuf + kTileH * kTilePitch + 16);
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
    const int tx0 = (unit.y % is->tiles_x) * kTileW, ty0 = (unit.y / is->tiles_x) * kTileH;
    const int tw = min(kTileW, Wo - tx0), th = min(kTileH, Ho - ty0);
    if (threadIdx.x == 0) {
      const int xwa = m.ax * tx0 + m.bx, xwb = m.ax * (tx0 + tw - 1) + m.bx;
      const int ywa = m.ay * ty0 + m.by, ywb = m.ay * (ty0 + th - 1) + m.by;
      const double xw0 = min(xwa, xwb), xw1 = max(xwa, xwb), yw0 = min(ywa, ywb), yw1 = max(ywa, ywb);
      const double* A = is->A;
      double lx = 1e300, hx = -1e300, ly = 1e300, hy = -1e300;
      for (int c = 0; c < 4; ++c) {
        const double xw = (c & 1) ? xw1 : xw0, yw = (c & 2) ? yw1 : yw0;
        const double sx = fma(A[0], xw, fma(A[1], yw, A[2]));
        const double sy = fma(A[3], xw, fma(A[4], yw, A[5]));
        lx = fmin(lx, sx); hx = fmax(hx, sx); ly = fmin(ly, sy); hy = fmax(hy, sy);
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
      *tg = t;
    }
    __syncthreads();
    const TileGeom t = *tg;
    const uint8_t* simg = a.src + sd.offset;
    if (t.staged) {
      // pass A: 16-pixel interior runs with 16-byte loads
      const int nvi = (t.ci1 - t.ci0) >> 4;
      if (nvi > 0) {
        const uint32_t magic = 0xffffffffu / (uint32_t)nvi + 1u;
        for (int it = threadIdx.x; it < t.fh * nvi; it += kAfThreads) {
          const int r = nvi == 1 ? it : (int)__umulhi((uint32_t)it, magic);
          const int c = t.ci0 + ((it - r * nvi) << 4);
          bool row_in;
          const int ry = border_idx(t.fy0 + r, Hs, reflect, row_in);
          uint32_t* d = stage + r * t.S + c;
          if (row_in) {
            const uint8_t* srow = simg + (size_t)ry * sd.pitch;
            uint32_t w[12];
            load_window<12>(srow + (size_t)(t.fx0 + c) * 3, srow, srow + (size_t)Ws * 3, w);
#pragma unroll
            for (int i = 0; i < 16; ++i) d[i] = rgbx_of(w, i);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) d[i] = a.fill;
          }
        }
      }
      // pass B: border columns + the interior tail, one pixel per thread
      const int tail = (t.ci1 - t.ci0) & 15;
      const int P = t.ci0 + tail + (t.fw - t.ci1);
      if (P > 0) {
        const uint32_t magic = 0xffffffffu / (uint32_t)P + 1u;
        for (int it = threadIdx.x; it < t.fh * P; it += kAfThreads) {
          const int r = P == 1 ? it : (int)__umulhi((uint32_t)it, magic);
          const int j = it - r * P;
          const int c = j < t.ci0 ? j : (j < t.ci0 + tail ? t.ci0 + 16 * nvi + (j - t.ci0)
                                                          : t.ci1 + (j - t.ci0 - tail));
          bool row_in, col_in;
          const int ry = border_idx(t.fy0 + r, Hs, reflect, row_in);
          const int rx = border_idx(t.fx0 + c, Ws, reflect, col_in);
          stage[r * t.S + c] = (row_in && col_in) ? fetch_rgb(simg + (size_t)ry * sd.pitch, rx) : a.fill;
        }
      }
      if (has_mask) {
        const uint8_t* smk = a.msrc + a.msdesc[img].offset;
        const int mpitch = a.msdesc[img].pitch;
        const uint32_t magic = 0xffffffffu / (uint32_t)t.fw + 1u;
        for (int it = threadIdx.x; it < t.fh * t.fw; it += kAfThreads) {
          const int r = t.fw == 1 ? it : (int)__umulhi((uint32_t)it, magic);
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
    uint8_t* dbase = nullptr;
    int dpitch = 0;
    if (!normalize) {
      const alb_image_desc dd = a.ddesc[img];
      dbase = a.dst + dd.offset;
      dpitch = dd.pitch;
    }
    int xw[2];
    float dxl[2];
    int cur_cy[2] = {-0x7fffffff, -0x7fffffff};
    int aix[2] = {0, 0}, aiy[2] = {0, 0};
    float afx[2] = {0.f, 0.f}, afy[2] = {0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      xw[j] = m.ax * min(tx0 + lane + 32 * j, Wo - 1) + m.bx;
      dxl[j] = (float)(xw[j] & 15);
    }
    for (int i = 0; i < kRowsPerWarp; ++i) {
      const int row = warp * kRowsPerWarp + i;
      if (row >= th) break;
      const int yo = ty0 + row;
      const int yw = m.ay * yo + m.by;
      const float dyl = (float)(yw & 15);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = lane + 32 * j;
        if (c >= tw) continue;
        if ((yw >> 4) != cur_cy[j]) {  // fp64 anchor of this column's 16x16 cell
          cur_cy[j] = yw >> 4;
          const double xa = (double)((xw[j] >> 4) * 16), ya = (double)(cur_cy[j] * 16);
          const double sx = fma(A[0], xa, fma(A[1], ya, A[2]));
          const double sy = fma(A[3], xa, fma(A[4], ya, A[5]));
          const double flx = floor(sx), fly = floor(sy);
          aix[j] = (int)flx; aiy[j] = (int)fly;
          afx[j] = (float)(sx - flx); afy[j] = (float)(sy - fly);
        }
        const float lx = fmaf(A0f, dxl[j], fmaf(A1f, dyl, afx[j]));
        const float ly = fmaf(A3f, dxl[j], fmaf(A4f, dyl, afy[j]));
        uint32_t r, g, b;
        if (nearest) {
          const int qx = aix[j] + (int)floorf(lx + 0.5f), qy = aiy[j] + (int)floorf(ly + 0.5f);
          uint32_t tt;
          if (t.staged) {
            tt = stage[(qy - t.fy0) * t.S + (qx - t.fx0)];
          } else {
            bool ri, ci;
            const int yy = border_idx(qy, Hs, reflect, ri), xx = border_idx(qx, Ws, reflect, ci);
            tt = (ri && ci) ? fetch_rgb(simg + (size_t)yy * sd.pitch, xx) : a.fill;
          }
          r = tt & 0xff; g = (tt >> 8) & 0xff; b = (tt >> 16) & 0xff;
        } else {
          const float flx = floorf(lx), fly = floorf(ly);
          const float fx = lx - flx, fy = ly - fly;
          const int qx = aix[j] + (int)flx, qy = aiy[j] + (int)fly;
          uint32_t t00, t10, t01, t11;
          if (t.staged) {
            const uint32_t* p = stage + (qy - t.fy0) * t.S + (qx - t.fx0);
            t00 = p[0]; t10 = p[1]; t01 = p[t.S]; t11 = p[t.S + 1];
          } else {
            auto tap = [&](int px, int py) -> uint32_t {
              bool ri, ci;
              const int yy = border_idx(py, Hs, reflect, ri), xx = border_idx(px, Ws, reflect, ci);
              return (ri && ci) ? fetch_rgb(simg + (size_t)yy * sd.pitch, xx) : a.fill;
            };
            t00 = tap(qx, qy); t10 = tap(qx + 1, qy); t01 = tap(qx, qy + 1); t11 = tap(qx + 1, qy + 1);
          }
          const uint32_t px = bilerp_rgbx(t00, t10, t01, t11, fx, fy);
          r = px & 0xff; g = (px >> 8) & 0xff; b = (px >> 16) & 0xff;
        }
        apply_stages_t<kOne>(x, sm, lane, r, g, b);
        if (normalize) {
          const size_t plane = (size_t)Ho * Wo;
          float* o = a.nchw + (size_t)img * 3 * plane + (size_t)yo * Wo + tx0 + c;
          const float* nl = a.tab.norm_lut;
          __stcs(o, nl[r]);
          __stcs(o + plane, nl[256 + g]);
          __stcs(o + 2 * plane, nl[512 + b]);
        } else {
          uint8_t* tb = tilebuf + row * kTilePitch + 3 * c;
          tb[0] = (uint8_t)r;
          tb[1] = (uint8_t)g;
          tb[2] = (uint8_t)b;
        }
        if (has_mask) {
          const int qx = aix[j] + (int)floorf(lx + 0.5f), qy = aiy[j] + (int)floorf(ly + 0.5f);
          uint8_t v;
          if (t.staged) {
            v = mstage[(qy - t.fy0) * t.Sm + (qx - t.fx0)];
          } else {
            bool ri, ci;
            const int yy = border_idx(qy, Hs, reflect, ri), xx = border_idx(qx, Ws, reflect, ci);
            v = (ri && ci) ? a.msrc[a.msdesc[img].offset + (size_t)yy * a.msdesc[img].pitch + xx]
                           : (uint8_t)a.mask_fill;
          }
          const alb_image_desc mdd = a.mddesc[img];
          a.mdst[mdd.offset + (size_t)yo * mdd.pitch + tx0 + c] = v;
        }
      }
    }
    if (!normalize) {  // the whole tile, aligned 16-byte stores
      __syncthreads();
      cta_copy_rows(dbase + (size_t)ty0 * dpitch + (size_t)tx0 * 3, dpitch, tilebuf, kTilePitch, th,
                    3 * tw, kAfThreads);
    }
  }
}

static size_t affine_smem(const StepArgs& a) {
  return (size_t)count_lut_stages(a) * kLutWords * 4 + sizeof(ImgState) + sizeof(TileGeom) +
         kTileH * kTilePitch + 16 + (size_t)a.unit_size * 4 +
         (a.mdst ? (size_t)a.unit_size : 0);
}

template <int kOne, bool kGeneric>
static void launch_affine_v(const StepArgs& a, size_t smem, cudaStream_t s) {
  const int grid = persistent_grid((const void*)k_affine<kOne, kGeneric>, kAfThreads, smem, a.n_units);
  k_affine<kOne, kGeneric><<<grid, kAfThreads, smem, s>>>(a);
}

template <int kOne>
static void launch_affine_t(const StepArgs& a, size_t smem, cudaStream_t s) {
  const bool generic = a.interp == ALB_INTERP_NEAREST || a.mdst != nullptr || a.normalize;
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
