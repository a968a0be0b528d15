// rowgather.cu -- exact geometric ops (K2 HFlip, K3 VFlip / RandomCrop / Crop /
// PadToSize, and any chain of them) as ONE integer map per image:
//   out[y][x] = in[ay*y + by][ax*x + bx]  (ax, ay = +-1), fill outside the
//   valid rectangle (O2-O4).
// Each thread produces one 16-pixel block of an output row whose first byte is
// 16-byte aligned AND on a pixel boundary (16*C bytes = 1 or 3 uint4 stores).
// The 16 source pixels are fetched with aligned 16-byte loads and realigned in
// registers (funnel shifts); HFlip reverses pixel order with byte permutes.
#include "kernels.cuh"

namespace alb {

constexpr int kRgThreads = 256;

// reverse the 16 pixels held in w (C bytes each), compile-time byte gather
template <int C>
__device__ __forceinline__ void reverse_px(uint32_t (&w)[4 * C]) {
  uint32_t o[4 * C];
#pragma unroll
  for (int m = 0; m < 4 * C; ++m) {
    uint32_t r = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = 4 * m + b;
      const int s = C * (15 - j / C) + j % C;
      r |= ((w[s >> 2] >> ((s & 3) * 8)) & 0xffu) << (b * 8);
    }
    o[m] = r;
  }
#pragma unroll
  for (int m = 0; m < 4 * C; ++m) w[m] = o[m];
}

template <int C>
__global__ void __launch_bounds__(kRgThreads) k_rowgather(StepArgs a, uint32_t fill) {
  const int2 unit = a.units[blockIdx.x];
  const int img = unit.x;
  const alb_image_desc sd = C == 3 ? a.sdesc[img] : a.msdesc[img];
  const alb_image_desc dd = C == 3 ? a.ddesc[img] : a.mddesc[img];
  const uint8_t* sbase = C == 3 ? a.src : a.msrc;
  uint8_t* dbase = C == 3 ? a.dst : a.mdst;
  const int Wo = dd.width, Ho = dd.height, Ws = sd.width;
  const Map1 m = compose_exact(a.ops, a.tab, img, a.slot0, a.slot1, Wo, Ho);
  const int y0 = unit.y * a.unit_size;
  const int y1 = min(Ho, y0 + a.unit_size);
  const int nbmax = 2 + Wo / 16;
  const int items = (y1 - y0) * nbmax;
  for (int it = threadIdx.x; it < items; it += kRgThreads) {
    const int y = y0 + it / nbmax;
    const int k = it % nbmax - 1;
    uint8_t* drow = dbase + dd.offset + (size_t)y * dd.pitch;
    const int pa = first_aligned_px_offset<C>((uintptr_t)drow) / C;
    const int xb = pa + 16 * k;
    if (xb + 16 <= 0 || xb >= Wo) continue;
    uint32_t w[4 * C];
    const bool row_ok = y >= m.vy0 && y < m.vy1;
    if (row_ok) {
      const int sy = m.ay * y + m.by;
      const uint8_t* srow = sbase + sd.offset + (size_t)sy * sd.pitch;
      const int sx_lo = m.ax > 0 ? xb + m.bx : m.bx - (xb + 15);
      load_window<4 * C>(srow + (ptrdiff_t)sx_lo * C, srow, srow + (size_t)Ws * C, w);
      if (m.ax < 0) reverse_px<C>(w);
      if (xb < m.vx0 || xb + 16 > m.vx1) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int x = xb + i;
          if (x < m.vx0 || x >= m.vx1) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
              const int j = C * i + c;
              const uint32_t f = (fill >> (8 * c)) & 0xffu;
              w[j >> 2] = (w[j >> 2] & ~(0xffu << ((j & 3) * 8))) | (f << ((j & 3) * 8));
            }
          }
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16 * C; ++j) {
        const uint32_t f = (fill >> (8 * (j % C))) & 0xffu;
        if ((j & 3) == 0) w[j >> 2] = 0;
        w[j >> 2] |= f << ((j & 3) * 8);
      }
    }
    uint8_t* dp = drow + (ptrdiff_t)xb * C;
    if (xb >= 0 && xb + 16 <= Wo) {
      uint4* d4 = reinterpret_cast<uint4*>(dp);
#pragma unroll
      for (int v = 0; v < C; ++v) __stcs(d4 + v, make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]));
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int x = xb + i;
        if (x >= 0 && x < Wo) {
#pragma unroll
          for (int c = 0; c < C; ++c) dp[C * i + c] = (uint8_t)byte_of(w, C * i + c);
        }
      }
    }
  }
}

void launch_rowgather(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  if (a.channels == 3)
    k_rowgather<3><<<a.n_units, kRgThreads, 0, s>>>(a, a.fill);
  else
    k_rowgather<1><<<a.n_units, kRgThreads, 0, s>>>(a, a.mask_fill);
}

}  // namespace alb
