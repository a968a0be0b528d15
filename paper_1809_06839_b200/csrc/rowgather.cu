// rowgather.cu -- exact geometric ops (K2 HFlip, K3 VFlip / RandomCrop / Crop /
// PadToSize, and any chain of them) as ONE integer map per image:
//   out[y][x] = in[ay*y + by][ax*x + bx]  (ax, ay = +-1), fill outside the
//   valid rectangle (O2-O4).
// Each thread produces one 16-pixel block of an output row whose first byte is
// 16-byte aligned AND on a pixel boundary (16*C bytes = 1 or 3 uint4 stores).
// The 16 source pixels are fetched with aligned 16-byte loads and realigned in
// registers (funnel shifts); HFlip reverses pixel order with byte permutes.
#include "stages.cuh"

namespace alb {

constexpr int kRgThreads = 256;

// reverse the 16 pixels held in w (C bytes each): every output word gathers
// its 4 bytes from <= 3 source words with one or two byte permutes whose
// selectors fold to constants after unrolling
template <int C>
__device__ __forceinline__ void reverse_px(uint32_t (&w)[4 * C]) {
  uint32_t o[4 * C];
#pragma unroll
  for (int m = 0; m < 4 * C; ++m) {
    int sb[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = 4 * m + b;
      sb[b] = C * (15 - j / C) + j % C;
    }
    int wa = sb[0] >> 2, wb = sb[0] >> 2;
#pragma unroll
    for (int b = 1; b < 4; ++b) {
      wa = min(wa, sb[b] >> 2);
      wb = max(wb, sb[b] >> 2);
    }
    if (wb - wa <= 1) {
      uint32_t sel = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) sel |= (uint32_t)(((sb[b] >> 2) - wa) * 4 + (sb[b] & 3)) << (4 * b);
      o[m] = __byte_perm(w[wa], w[wa + 1 < 4 * C ? wa + 1 : wa], sel);
    } else {  // three source words: (wa, wa+1) first, then merge word wa+2
      uint32_t s1 = 0, s2 = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int q = (sb[b] >> 2) - wa;
        s1 |= (uint32_t)(q <= 1 ? q * 4 + (sb[b] & 3) : 0) << (4 * b);
        s2 |= (uint32_t)(q == 2 ? 4 + (sb[b] & 3) : b) << (4 * b);
      }
      o[m] = __byte_perm(__byte_perm(w[wa], w[wa + 1], s1), w[wa + 2], s2);
    }
  }
#pragma unroll
  for (int m = 0; m < 4 * C; ++m) w[m] = o[m];
}

// One CTA per (image, band of rows) unit (the loop also serves persistent
// launches); the per-image integer map is composed once per image change.  Item = (row, 16-pixel block whose first
// destination byte is 16-byte aligned and on a pixel boundary).
template <int C>
__global__ void __launch_bounds__(kRgThreads) k_rowgather(StepArgs a, uint32_t fill) {
  __shared__ Map1 smap;
  int u0, u1;
  unit_range(a.n_units, u0, u1);
  int cur_img = -1;
  Map1 m{};
  int Wo = 0, Ho = 0, Ws = 0, nbmax = 0;
  uint32_t mnb = 0;
  alb_image_desc sd{}, dd{};
  const uint8_t* sbase = C == 3 ? a.src : a.msrc;
  uint8_t* dbase = C == 3 ? a.dst : a.mdst;
  for (int u = u0; u < u1; ++u) {
    const int2 unit = a.units[u];
    const int img = unit.x;
    if (img != cur_img) {
      __syncthreads();
      sd = C == 3 ? a.sdesc[img] : a.msdesc[img];
      dd = C == 3 ? a.ddesc[img] : a.mddesc[img];
      Wo = dd.width; Ho = dd.height; Ws = sd.width;
      if (threadIdx.x == 0) smap = compose_exact(a.ops, a.tab, img, a.slot0, a.slot1, Wo, Ho);
      nbmax = 2 + Wo / 16;
      mnb = magic_of((uint32_t)nbmax);
      __syncthreads();
      m = smap;
      cur_img = img;
    }
    const int y0 = unit.y * a.unit_size;
    const int y1 = min(Ho, y0 + a.unit_size);
    const int items = (y1 - y0) * nbmax;
    for (int it = threadIdx.x; it < items; it += kRgThreads) {
      const int yy = fdiv(it, mnb);
      const int y = y0 + yy;
      const int k = it - yy * nbmax - 1;
      uint8_t* drow = dbase + dd.offset + (size_t)y * dd.pitch;
      const int o = (int)((uintptr_t)drow & 15);
      const int pa = C == 3 ? (11 * (16 - o)) & 15 : (16 - o) & 15;  // first aligned pixel
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
}

void launch_rowgather(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  // one CTA per unit (unit_range gives each CTA exactly its own unit)
  if (a.channels == 3)
    k_rowgather<3><<<a.n_units, kRgThreads, 0, s>>>(a, a.fill);
  else
    k_rowgather<1><<<a.n_units, kRgThreads, 0, s>>>(a, a.mask_fill);
}

}  // namespace alb
