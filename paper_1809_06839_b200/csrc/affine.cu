// affine.cu -- K4 Rotate / ShiftScaleRotate (O7) with fused post
// ops (K10: RandomCrop / Crop / flips on the output coordinates), the
// pointwise stage chain, Normalize output and the nearest-neighbour mask.
//
// Inverse map per warp-output pixel (xw, yw):
//   x_s = cx + (cos*(xw-cx-tx) - sin*(yw-cy-ty)) / s,  likewise y_s,
// written as x_s = A0*xw + A1*yw + A2 with the coefficients formed in fp64.
// Coordinates use an fp64 ANCHOR per 16-pixel group of warp-output columns
// (xw & ~15, yw) plus an fp32 local offset (xw & 15)*A0: error < 2e-6 px,
// and the value of a pixel depends only on its warp-output coordinates, so the
// fused cfg5 kernel equals the unfused Rotate/SSR kernel bit for bit.
// Bilinear blend in fp32; border per tap (reflect-101 or constant, R7).
//
// Work unit = (image, band of output rows); each thread produces aligned
// 16-pixel blocks.  The source footprint of the band is staged in shared
// memory as RGBx words when it fits; taps outside the image resolve the border
// per tap.
#include "stages.cuh"

namespace alb {

constexpr int kAfThreads = 256;
constexpr int kAfBand = 16;

struct AfCoef {
  double A[6];
};

__device__ __forceinline__ AfCoef af_coef(const StepArgs& a, int img) {
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
  AfCoef c;
  const double ux = __dadd_rn(cx, tx), uy = __dadd_rn(cy, ty);
  c.A[0] = cs / s;
  c.A[1] = -sn / s;
  c.A[2] = cx - (cs * ux - sn * uy) / s;
  c.A[3] = sn / s;
  c.A[4] = cs / s;
  c.A[5] = cy - (sn * ux + cs * uy) / s;
  return c;
}

__device__ __forceinline__ uint32_t fetch_rgb(const uint8_t* base, int pitch, int x, int y) {
  const uint8_t* p = base + (size_t)y * pitch + 3 * x;
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16);
}

__global__ void __launch_bounds__(kAfThreads) k_affine(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int2 unit = a.units[blockIdx.x];
  const int img = unit.x;
  const int lane = threadIdx.x & 31;
  const alb_image_desc sd = a.sdesc[img];
  const int Ws = sd.width, Hs = sd.height;
  const int Wo = a.normalize ? a.out_w : a.ddesc[img].width;
  const int Ho = a.normalize ? a.out_h : a.ddesc[img].height;
  const Map1 m = compose_exact(a.ops, a.tab, img, a.slot0 + 1, a.slot1, Wo, Ho);
  const bool warp_on = fired_of(a.tab, img, a.slot0);
  AfCoef cf;
  if (warp_on) {
    cf = af_coef(a, img);
  } else {
    cf.A[0] = 1; cf.A[1] = 0; cf.A[2] = 0; cf.A[3] = 0; cf.A[4] = 1; cf.A[5] = 0;
  }
  const float a0f = (float)cf.A[0], a3f = (float)cf.A[3];
  const int y0 = unit.y * kAfBand;
  const int y1 = min(Ho, y0 + kAfBand);
  const bool reflect = a.border == ALB_BORDER_REFLECT_101;
  const bool nearest = a.interp == ALB_INTERP_NEAREST;

  StageCtx x;
  load_stages(a, img, sm, x, kAfThreads);
  uint32_t* stage = sm + x.n_lut * kLutWords;

  // footprint of the band in source coordinates: map the corners of the
  // band's warp-output bounding box (post map is a +-1 integer map)
  int fx0, fx1, fy0, fy1;
  {
    const int xa = m.ax * 0 + m.bx, xb2 = m.ax * (Wo - 1) + m.bx;
    const int ya = m.ay * y0 + m.by, yb = m.ay * (y1 - 1) + m.by;
    const double xw0 = min(xa, xb2), xw1 = max(xa, xb2), yw0 = min(ya, yb), yw1 = max(ya, yb);
    double lx = 1e30, hx = -1e30, ly = 1e30, hy = -1e30;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double xw = (c & 1) ? xw1 : xw0, yw = (c & 2) ? yw1 : yw0;
      const double xs = cf.A[0] * xw + cf.A[1] * yw + cf.A[2];
      const double ys = cf.A[3] * xw + cf.A[4] * yw + cf.A[5];
      lx = fmin(lx, xs); hx = fmax(hx, xs); ly = fmin(ly, ys); hy = fmax(hy, ys);
    }
    fx0 = (int)floor(lx) - 1; fx1 = (int)floor(hx) + 2;
    fy0 = (int)floor(ly) - 1; fy1 = (int)floor(hy) + 2;
  }
  const int fw = fx1 - fx0 + 1, fh = fy1 - fy0 + 1;
  const bool staged = a.unit_size > 0 && (long long)fw * fh <= a.unit_size && fw > 0 && fh > 0;
  const uint32_t fillpx = a.fill;
  if (staged) {
    // stage [fx0,fx1] x [fy0,fy1] with the border resolved per staged pixel
    const int per_row = (fw + 15) / 16;
    for (int it = threadIdx.x; it < fh * per_row; it += kAfThreads) {
      const int r = it / per_row, c16 = (it % per_row) * 16;
      const int sy = fy0 + r;
      int ry = sy;
      bool row_in = sy >= 0 && sy < Hs;
      if (!row_in && reflect) { ry = reflect101(sy, Hs); row_in = true; }
      uint32_t* d = stage + r * fw + c16;
      const int sx0 = fx0 + c16;
      const uint8_t* srow = a.src + sd.offset + (size_t)ry * sd.pitch;
      if (row_in && sx0 >= 0 && sx0 + 16 <= Ws) {
        uint32_t w[12];
        load_window<12>(srow + (size_t)sx0 * 3, srow, srow + (size_t)Ws * 3, w);
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (c16 + i < fw) d[i] = byte_of(w, 3 * i) | (byte_of(w, 3 * i + 1) << 8) | (byte_of(w, 3 * i + 2) << 16);
      } else {
        for (int i = 0; i < 16 && c16 + i < fw; ++i) {
          const int sx = sx0 + i;
          uint32_t v = fillpx;
          if (row_in) {
            if (sx >= 0 && sx < Ws) v = fetch_rgb(srow, 0, sx, 0);
            else if (reflect) v = fetch_rgb(srow, 0, reflect101(sx, Ws), 0);
          }
          d[i] = v;
        }
      }
    }
  }
  __syncthreads();

  const uint8_t* sbase = a.src + sd.offset;
  auto tap = [&](int tx, int ty) -> uint32_t {
    if (staged) return stage[(ty - fy0) * fw + (tx - fx0)];
    if (tx >= 0 && tx < Ws && ty >= 0 && ty < Hs) return fetch_rgb(sbase, sd.pitch, tx, ty);
    if (!reflect) return fillpx;
    return fetch_rgb(sbase, sd.pitch, reflect101(tx, Ws), reflect101(ty, Hs));
  };

  const int nbmax = 2 + Wo / 16;
  const int items = (y1 - y0) * nbmax;
  for (int it = threadIdx.x; it < items; it += kAfThreads) {
    const int yy = y0 + it / nbmax;
    const int k = it % nbmax - 1;
    int xb;
    uint8_t* drow = nullptr;
    if (a.normalize) {
      xb = 16 * k;
    } else {
      const alb_image_desc dd = a.ddesc[img];
      drow = a.dst + dd.offset + (size_t)yy * dd.pitch;
      xb = first_aligned_px_offset<3>((uintptr_t)drow) / 3 + 16 * k;
    }
    if (xb + 16 <= 0 || xb >= Wo) continue;
    const int yw = m.ay * yy + m.by;
    int cur_g = -0x7fffffff;
    double ixd = 0, iyd = 0;
    float fxa = 0.f, fya = 0.f;
    uint32_t px[48];
#pragma unroll 4
    for (int i = 0; i < 16; ++i) {
      const int xo = min(max(xb + i, 0), Wo - 1);
      const int xw = m.ax * xo + m.bx;
      const int gq = xw >> 4;
      if (gq != cur_g) {  // fp64 anchor of this 16-column group
        cur_g = gq;
        const double xa = (double)(gq * 16);
        const double sx = fma(cf.A[0], xa, fma(cf.A[1], (double)yw, cf.A[2]));
        const double sy = fma(cf.A[3], xa, fma(cf.A[4], (double)yw, cf.A[5]));
        ixd = floor(sx); iyd = floor(sy);
        fxa = (float)(sx - ixd); fya = (float)(sy - iyd);
      }
      const float li = (float)(xw & 15);
      const float lx = fmaf(li, a0f, fxa), ly = fmaf(li, a3f, fya);
      uint32_t ch[3];
      if (nearest) {
        const int tx = (int)ixd + (int)floorf(lx + 0.5f), ty = (int)iyd + (int)floorf(ly + 0.5f);
        const uint32_t t = tap(tx, ty);
        ch[0] = t & 0xff; ch[1] = (t >> 8) & 0xff; ch[2] = (t >> 16) & 0xff;
      } else {
        const float flx = floorf(lx), fly = floorf(ly);
        const float fx = lx - flx, fy = ly - fly;
        const int tx = (int)ixd + (int)flx, ty = (int)iyd + (int)fly;
        const uint32_t t00 = tap(tx, ty), t10 = tap(tx + 1, ty);
        const uint32_t t01 = tap(tx, ty + 1), t11 = tap(tx + 1, ty + 1);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float p00 = (float)((t00 >> (8 * c)) & 0xff), p10 = (float)((t10 >> (8 * c)) & 0xff);
          const float p01 = (float)((t01 >> (8 * c)) & 0xff), p11 = (float)((t11 >> (8 * c)) & 0xff);
          const float h0 = (1.f - fx) * p00 + fx * p10;
          const float h1 = (1.f - fx) * p01 + fx * p11;
          const float v = (1.f - fy) * h0 + fy * h1;
          ch[c] = (uint32_t)min(255, (int)floorf(v + 0.5f));
        }
      }
      apply_stages(a, x, sm, lane, ch[0], ch[1], ch[2]);
      px[3 * i] = ch[0]; px[3 * i + 1] = ch[1]; px[3 * i + 2] = ch[2];
    }
    if (a.normalize) {
      store_nchw(a, img, yy, xb, px, Wo, Ho);
    } else {
      uint32_t w[12];
#pragma unroll
      for (int q = 0; q < 12; ++q)
        w[q] = px[4 * q] | (px[4 * q + 1] << 8) | (px[4 * q + 2] << 16) | (px[4 * q + 3] << 24);
      store_block<3>(drow, xb, Wo, w);
    }
  }

  // mask: nearest with the same anchored coordinates, constant mask_fill
  if (a.mdst) {
    const alb_image_desc msd = a.msdesc[img];
    const alb_image_desc mdd = a.mddesc[img];
    const uint8_t* mb = a.msrc + msd.offset;
    for (int it = threadIdx.x; it < (y1 - y0) * Wo; it += kAfThreads) {
      const int yy = y0 + it / Wo, xo = it % Wo;
      const int xw = m.ax * xo + m.bx, yw = m.ay * yy + m.by;
      const int gq = xw >> 4;
      const double xa = (double)(gq * 16);
      const double sx = fma(cf.A[0], xa, fma(cf.A[1], (double)yw, cf.A[2]));
      const double sy = fma(cf.A[3], xa, fma(cf.A[4], (double)yw, cf.A[5]));
      const double ixd = floor(sx), iyd = floor(sy);
      const float li = (float)(xw & 15);
      const float lx = fmaf(li, a0f, (float)(sx - ixd)), ly = fmaf(li, a3f, (float)(sy - iyd));
      int tx = (int)ixd + (int)floorf(lx + 0.5f), ty = (int)iyd + (int)floorf(ly + 0.5f);
      uint8_t v = (uint8_t)a.mask_fill;
      if (tx >= 0 && tx < Ws && ty >= 0 && ty < Hs) {
        v = mb[(size_t)ty * msd.pitch + tx];
      } else if (reflect) {
        v = mb[(size_t)reflect101(ty, Hs) * msd.pitch + reflect101(tx, Ws)];
      }
      a.mdst[mdd.offset + (size_t)yy * mdd.pitch + xo] = v;
    }
  }
}

void launch_affine(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  const size_t smem = (size_t)count_lut_stages(a) * kLutWords * 4 + (size_t)a.unit_size * 4;
  cudaFuncSetAttribute(k_affine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_affine<<<a.n_units, kAfThreads, smem, s>>>(a);
}

}  // namespace alb
