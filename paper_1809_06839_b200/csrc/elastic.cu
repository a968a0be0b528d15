// elastic.cu -- K12 ElasticTransform (reading
// R32): per 32x32 output tile, the displacement field is rebuilt from the
// counter-based raw planes (no per-image field in HBM), blurred in fp64 and
// used to remap the image (and mask) from global memory.
//
//   raw  u, v = -1 + 2 u53(draw j), j = 1 + y W + x  (u) / 1 + H W + y W + x  (v)
//   bx   = sum_k w_k raw[y][refl(x + k)]   (ascending k, acc = fma(w_k, v, acc))
//   d    = alpha * sum_k w_k bx[refl(y + k)][x]
//   out  = sample(x + dx, y + dy)          (bilinear / nearest, constant or reflect-101)
//
// The weights w_k are computed once per plan on the host (libm exp, the same
// bits the oracle computes) and the blur runs in fp64 in the definition's order,
// so source coordinates are bit-identical to the oracle's; only the bilinear
// blend runs in fp32 (bilerp3).
//
// Work unit = (image, 32x32 output tile); one CTA (8 warps) per unit.
//   x pass: warp per halo row (32 + 2r rows), the row's 32 + 2r raw values in a
//           per-warp buffer, lane = output column;
//   y pass: thread per (row, column), 4 rows per thread;
//   remap:  thread per output pixel, taps from global memory (L1/L2 resident:
//           |d| stays far below alpha for smooth fields, so neighbouring tiles
//           share lines).
#include "stages.cuh"

namespace alb {

constexpr int kElT = 32;
constexpr int kElThreads = 256;
constexpr int kElWarps = kElThreads / 32;

size_t elastic_smem(int r) {
  const int hr = kElT + 2 * r;
  return (size_t)(2 * kElMaxR + 1) * 8            // weights
         + (size_t)kElWarps * hr * 8               // raw row per warp
         + (size_t)hr * kElT * 8                   // x-pass rows
         + (size_t)2 * kElT * kElT * 8;            // dx, dy
}

__device__ __forceinline__ double raw_uv(const StepArgs& a, uint32_t gi, int j) {
  return urange(-1.0, 1.0, draw_u(a.seed, gi, a.slot0, j));
}

__global__ void __launch_bounds__(kElThreads) k_elastic(StepArgs a) {
  extern __shared__ double esm[];
  const int r = a.g_r, hr = kElT + 2 * r;
  double* wgt = esm;
  double* rawb = wgt + (2 * kElMaxR + 1);
  double* bx = rawb + kElWarps * hr;
  double* dxy = bx + hr * kElT;  // [2][32][32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int2 unit = a.units[blockIdx.x];
  const int img = unit.x;
  const alb_image_desc sd = a.sdesc[img];
  const int W = sd.width, H = sd.height;
  const int x0 = (unit.y & 0xffff) * kElT, y0 = (unit.y >> 16) * kElT;
  const bool fired = fired_of(a.tab, img, a.slot0);
  if (fired) {
    for (int k = tid; k <= 2 * r; k += kElThreads) wgt[k] = a.gauss[k];
    __syncthreads();
    const uint32_t gi = a.first_image + (uint32_t)img;
    const int plane_j = W * H;
    double* rb = rawb + warp * hr;
    for (int plane = 0; plane < 2; ++plane) {
      const int j0 = 1 + plane * plane_j;
      // x pass over the halo rows
      for (int ry = warp; ry < hr; ry += kElWarps) {
        const int yy = reflect101(y0 - r + ry, H);
        const int jr = j0 + yy * W;
        for (int q = lane; q < hr; q += 32) rb[q] = raw_uv(a, gi, jr + reflect101(x0 - r + q, W));
        __syncwarp();
        double acc = 0.0;
        for (int k = 0; k <= 2 * r; ++k) acc = __fma_rn(wgt[k], rb[lane + k], acc);
        bx[ry * kElT + lane] = acc;
        __syncwarp();
      }
      __syncthreads();
      // y pass
      double* d = dxy + plane * kElT * kElT;
      for (int row = warp; row < kElT; row += kElWarps) {
        double acc = 0.0;
        for (int k = 0; k <= 2 * r; ++k) acc = __fma_rn(wgt[k], bx[(row + k) * kElT + lane], acc);
        d[row * kElT + lane] = __dmul_rn(a.alpha, acc);
      }
      __syncthreads();
    }
  }
  // remap
  const bool reflect = a.border == ALB_BORDER_REFLECT_101;
  const bool nearest = a.interp == ALB_INTERP_NEAREST;
  const uint8_t* simg = a.src + sd.offset;
  const alb_image_desc dd = a.ddesc[img];
  uint8_t* dimg = a.dst + dd.offset;
  const uint8_t* smk = a.mdst ? a.msrc + a.msdesc[img].offset : nullptr;
  const int mps = a.mdst ? a.msdesc[img].pitch : 0;
  uint8_t* dmk = a.mdst ? a.mdst + a.mddesc[img].offset : nullptr;
  const int mpd = a.mdst ? a.mddesc[img].pitch : 0;
  const int x = x0 + lane;
  for (int row = warp; row < kElT; row += kElWarps) {
    const int y = y0 + row;
    if (x >= W || y >= H) continue;
    double xs = (double)x, ys = (double)y;
    if (fired) {
      xs = __dadd_rn(xs, dxy[row * kElT + lane]);
      ys = __dadd_rn(ys, dxy[kElT * kElT + row * kElT + lane]);
    }
    const int xn = (int)floor(__dadd_rn(xs, 0.5)), yn = (int)floor(__dadd_rn(ys, 0.5));
    uint32_t v;
    if (nearest) {
      bool ix, iy;
      const int px = border_idx(xn, W, reflect, ix), py = border_idx(yn, H, reflect, iy);
      v = (ix && iy) ? fetch_rgb(simg + (size_t)py * sd.pitch, px) : a.fill;
    } else {
      const double fx0 = floor(xs), fy0 = floor(ys);
      const int xa = (int)fx0, ya = (int)fy0;
      const float2 f = make_float2((float)__dsub_rn(xs, fx0), (float)__dsub_rn(ys, fy0));
      uint32_t t[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        bool ix, iy;
        const int px = border_idx(xa + (q & 1), W, reflect, ix), py = border_idx(ya + (q >> 1), H, reflect, iy);
        t[q] = (ix && iy) ? fetch_rgb(simg + (size_t)py * sd.pitch, px) : a.fill;
      }
      uint32_t rr, gg, bb;
      bilerp3(t[0], t[1], t[2], t[3], f, rr, gg, bb);
      v = (rr & 0xffu) | ((gg & 0xffu) << 8) | ((bb & 0xffu) << 16);
    }
    uint8_t* o = dimg + (size_t)y * dd.pitch + 3 * x;
    o[0] = (uint8_t)v;
    o[1] = (uint8_t)(v >> 8);
    o[2] = (uint8_t)(v >> 16);
    if (dmk) {
      bool ix, iy;
      const int px = border_idx(xn, W, reflect, ix), py = border_idx(yn, H, reflect, iy);
      dmk[(size_t)y * mpd + x] = (ix && iy) ? smk[(size_t)py * mps + px] : (uint8_t)a.mask_fill;
    }
  }
}

void launch_elastic(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  const size_t smem = elastic_smem(a.g_r);
  persistent_grid((const void*)k_elastic, kElThreads, smem, a.n_units);  // smem attribute
  k_elastic<<<a.n_units, kElThreads, smem, s>>>(a);
}

}  // namespace alb
