// rowgather.cu -- exact geometric ops (K2 HFlip, K3 VFlip / RandomCrop / Crop /
// PadToSize, and any chain of them) as ONE integer map per image:
//   out[y][x] = in[ay*y + by][ax*x + bx]  (ax, ay = +-1), fill outside the
//   valid rectangle (O2-O4).
// Each thread produces one 16-pixel block of an output row whose first byte is
// 16-byte aligned AND on a pixel boundary (16*C bytes = 1 or 3 uint4 stores),
// or, for window steps, one 32-pixel block on a 32-byte boundary (3 256-bit
// stores, source from 256-bit loads).  Flip-only steps use k_rowflip (one
// warp per row, see there).
// The 16 source pixels are fetched with aligned 16-byte loads and realigned in
// registers (funnel shifts); HFlip reverses pixel order with byte permutes.
#include "stages.cuh"

namespace alb {

constexpr int kRgThreads = 256;

// reverse the 16 pixels held in w (C bytes each): every output word gathers
// its 4 bytes from <= 3 source words with one or two byte permutes whose
// selectors fold to constants after unrolling
template <int C, int NPX>
__device__ __forceinline__ void reverse_px(uint32_t (&w)[NPX * C / 4]) {
  constexpr int NW = NPX * C / 4;
  uint32_t o[NW];
#pragma unroll
  for (int m = 0; m < NW; ++m) {
    int sb[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = 4 * m + b;
      sb[b] = C * (NPX - 1 - j / C) + j % C;
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
      o[m] = __byte_perm(w[wa], w[wa + 1 < NW ? wa + 1 : wa], sel);
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
  for (int m = 0; m < NW; ++m) w[m] = o[m];
}

// NW words of a byte window starting at p (any alignment) from 32-byte aligned
// 256-bit loads; loads that do not overlap [lo, hi) read zeros
template <int NW>
__device__ __forceinline__ void load_window32(const uint8_t* __restrict__ p, const uint8_t* lo, const uint8_t* hi,
                                              uint32_t (&w)[NW]) {
  constexpr int NV = (4 * NW + 31 + 31) / 32;
  const uintptr_t a = (uintptr_t)p;
  const uint8_t* base = (const uint8_t*)(a & ~(uintptr_t)31);
  const int sh = (int)(a & 31);
  uint32_t r[NV * 8];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const uint8_t* q = base + 32 * v;
    uint32_t x[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (q < hi && q + 32 > lo) ld256_nc(q, x);
#pragma unroll
    for (int i = 0; i < 8; ++i) r[8 * v + i] = x[i];
  }
  const int qw = sh >> 2, kb = (sh & 3) * 8;
  uint32_t t1[NV * 8 - 1];
#pragma unroll
  for (int i = 0; i < NV * 8 - 1; ++i) t1[i] = (qw & 1) ? r[i + 1] : r[i];
  uint32_t t2[NV * 8 - 3];
#pragma unroll
  for (int i = 0; i < NV * 8 - 3; ++i) t2[i] = (qw & 2) ? t1[i + 2] : t1[i];
  uint32_t t3[NW + 1];
#pragma unroll
  for (int i = 0; i < NW + 1; ++i) t3[i] = (qw & 4) ? t2[i + 4] : t2[i];
#pragma unroll
  for (int i = 0; i < NW; ++i) w[i] = __funnelshift_r(t3[i], t3[i + 1], kb);
}

// One CTA per (image, band of rows) unit (the loop also serves persistent
// launches); the per-image integer map is composed once per image change.  Item = (row, 16-pixel block whose first
// destination byte is 16-byte aligned and on a pixel boundary).
template <int C, int NPX>
__global__ void __launch_bounds__(kRgThreads, 6) k_rowgather(StepArgs a, uint32_t fill) {
  constexpr int NW = NPX * C / 4, AL = NPX == 32 ? 32 : 16;  // words per item, store alignment
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
      if (threadIdx.x == 0) {
        if (a.self_sample) {  // the only step: draw this image's params here (no K0)
          SelfTables st;
          const Tables t = self_sample_tables(a, img, st);
          smap = compose_exact(a.ops, t, 0, a.slot0, a.slot1, Wo, Ho);
        } else {
          smap = compose_exact(a.ops, a.tab, img, a.slot0, a.slot1, Wo, Ho);
        }
      }
      nbmax = 2 + Wo / NPX;
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
      const int o = (int)((uintptr_t)drow & (AL - 1));
      const int pa = C == 3 ? (11 * (AL - o)) & (AL - 1) : (AL - o) & (AL - 1);  // first aligned pixel
      const int xb = pa + NPX * k;
      if (xb + NPX <= 0 || xb >= Wo) continue;
      uint32_t w[NW];
      const bool row_ok = y >= m.vy0 && y < m.vy1;
      if (row_ok) {
        const int sy = m.ay * y + m.by;
        const uint8_t* srow = sbase + sd.offset + (size_t)sy * sd.pitch;
        const int sx_lo = m.ax > 0 ? xb + m.bx : m.bx - (xb + NPX - 1);
        if constexpr (NPX == 32) load_window32<NW>(srow + (ptrdiff_t)sx_lo * C, srow, srow + (size_t)Ws * C, w);
        else load_window<NW>(srow + (ptrdiff_t)sx_lo * C, srow, srow + (size_t)Ws * C, w);
        if (m.ax < 0) reverse_px<C, NPX>(w);
        if (xb < m.vx0 || xb + NPX > m.vx1) {
#pragma unroll
          for (int i = 0; i < NPX; ++i) {
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
        for (int j = 0; j < NPX * C; ++j) {
          const uint32_t f = (fill >> (8 * (j % C))) & 0xffu;
          if ((j & 3) == 0) w[j >> 2] = 0;
          w[j >> 2] |= f << ((j & 3) * 8);
        }
      }
      uint8_t* dp = drow + (ptrdiff_t)xb * C;
      if (xb >= 0 && xb + NPX <= Wo) {
        if constexpr (NPX == 32) {
#pragma unroll
          for (int v = 0; v < C; ++v) {
            uint32_t q[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) q[i] = w[8 * v + i];
            st256_cs(dp + 32 * v, q);
          }
        } else {
          uint4* d4 = reinterpret_cast<uint4*>(dp);
#pragma unroll
          for (int v = 0; v < C; ++v) __stcs(d4 + v, make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]));
        }
      } else {
#pragma unroll
        for (int i = 0; i < NPX; ++i) {
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

// Flips only (any chain of HFlip / VFlip: the map's valid rectangle is the
// whole output, no fill).  One warp per output row: the row's 16-pixel blocks
// whose first byte is 16-byte aligned go one per lane (three aligned 16-byte
// loads + one more when the source run is misaligned, funnel-shift realign,
// compile-time byte-permute reversal, C aligned 16-byte streaming stores); the
// row's unaligned head and tail bytes (< 16 pixels each) are copied one byte
// per lane by the whole warp, so no lane runs a divergent byte loop.
template <int C>
#ifndef ALB_FLIP_MINB
#define ALB_FLIP_MINB 6  // 40 registers, 6 CTAs / SM: more rows in flight (measured 0.296 vs 0.32-0.35 ms)
#endif
__global__ void __launch_bounds__(kRgThreads, ALB_FLIP_MINB) k_rowflip(StepArgs a) {
  constexpr int NW = 4 * C, NV = C + 1;  // words per block, 16-byte loads per block
  __shared__ Map1 smap;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int2 unit = a.units[blockIdx.x];
  const int img = unit.x;
  const alb_image_desc sd = C == 3 ? a.sdesc[img] : a.msdesc[img];
  const alb_image_desc dd = C == 3 ? a.ddesc[img] : a.mddesc[img];
  const int Wo = dd.width, Ho = dd.height;
  if (threadIdx.x == 0) {
    if (a.self_sample) {  // the only step: draw this image's params here (no K0)
      SelfTables st;
      const Tables t = self_sample_tables(a, img, st);
      smap = compose_exact(a.ops, t, 0, a.slot0, a.slot1, Wo, Ho);
    } else {
      smap = compose_exact(a.ops, a.tab, img, a.slot0, a.slot1, Wo, Ho);
    }
  }
  __syncthreads();
  const Map1 m = smap;
  const uint8_t* sbase = (C == 3 ? a.src : a.msrc) + sd.offset;
  uint8_t* dbase = (C == 3 ? a.dst : a.mdst) + dd.offset;
  const int y0 = unit.y * a.unit_size, y1 = min(Ho, y0 + a.unit_size);
  for (int y = y0 + warp; y < y1; y += kRgThreads / 32) {
    uint8_t* drow = dbase + (size_t)y * dd.pitch;
    const uint8_t* srow = sbase + (size_t)(m.ay * y + m.by) * sd.pitch;
    const int o = (int)((uintptr_t)drow & 15);
    const int pa = min(Wo, C == 3 ? (11 * (16 - o)) & 15 : (16 - o) & 15);  // first aligned pixel
    const int nfull = (Wo - pa) >> 4;
    for (int k = lane; k < nfull; k += 32) {
      const int xb = pa + 16 * k;
      const int sx_lo = m.ax > 0 ? xb + m.bx : m.bx - (xb + 15);
      const uintptr_t p = (uintptr_t)(srow + (ptrdiff_t)sx_lo * C);
      const uint4* q = reinterpret_cast<const uint4*>(p & ~(uintptr_t)15);
      const int sh = (int)(p & 15);
      uint32_t r[4 * NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        uint4 x = make_uint4(0, 0, 0, 0);
        if (v < NV - 1 || sh != 0) x = __ldg(q + v);  // the last vector only when the run is misaligned
        r[4 * v] = x.x; r[4 * v + 1] = x.y; r[4 * v + 2] = x.z; r[4 * v + 3] = x.w;
      }
      const int qw = sh >> 2, kb = (sh & 3) * 8;
      uint32_t t1[4 * NV - 1], t2[NW + 1], w[NW];
#pragma unroll
      for (int i = 0; i < 4 * NV - 1; ++i) t1[i] = (qw & 1) ? r[i + 1] : r[i];
#pragma unroll
      for (int i = 0; i < NW + 1; ++i) t2[i] = (qw & 2) ? t1[i + 2] : t1[i];
#pragma unroll
      for (int i = 0; i < NW; ++i) w[i] = __funnelshift_r(t2[i], t2[i + 1], kb);
      if (m.ax < 0) reverse_px<C, 16>(w);
      uint4* d4 = reinterpret_cast<uint4*>(drow + (ptrdiff_t)xb * C);
#pragma unroll
      for (int v = 0; v < C; ++v) __stcs(d4 + v, make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]));
    }
    const int nh = pa * C, xt = pa + 16 * nfull, nb = nh + (Wo - xt) * C;
    for (int t = lane; t < nb; t += 32) {
      const int b = t < nh ? t : xt * C + (t - nh);
      const int x = C == 3 ? b / 3 : b;
      drow[b] = srow[(m.ax * x + m.bx) * C + (b - x * C)];
    }
  }
}

void launch_rowgather(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  // one CTA per unit (unit_range gives each CTA exactly its own unit)
  // 32-pixel items with 256-bit accesses for window steps (crop / pad: few
  // loads per store; measured: pad 0.455 -> 0.404 ms); 16-pixel items with
  // 16-byte loads where every output byte is read from a shifted source (flips:
  // 40 vs 64 registers, measured 0.43 vs 0.55 ms)
  if (a.rg_wide == 2) {
    if (a.channels == 3) k_rowflip<3><<<a.n_units, kRgThreads, 0, s>>>(a);
    else k_rowflip<1><<<a.n_units, kRgThreads, 0, s>>>(a);
  } else if (a.channels == 3 && a.rg_wide)
    k_rowgather<3, 32><<<a.n_units, kRgThreads, 0, s>>>(a, a.fill);
  else if (a.channels == 3)
    k_rowgather<3, 16><<<a.n_units, kRgThreads, 0, s>>>(a, a.fill);
  else
    k_rowgather<1, 16><<<a.n_units, kRgThreads, 0, s>>>(a, a.mask_fill);
}

}  // namespace alb
