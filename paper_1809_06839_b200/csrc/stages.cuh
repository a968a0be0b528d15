// stages.cuh -- pointwise stage chain (LUT / Equalize LUT / HSV / gray) shared
// by the pointwise, resample and affine kernels so fused and unfused paths
// execute the same arithmetic.
#pragma once
#include "kernels.cuh"

namespace alb {

constexpr int kLutWords = 3 * 64 * 32;  // one lane-replicated LUT stage (24 KB)

struct StageData {
  float dh, ds, dv;
  int on;
};

struct StageCtx {
  StageData sd[kMaxStages];
  int n_lut;
};

__device__ __forceinline__ uint32_t lut_look(const uint32_t* __restrict__ sm, int cbase,
                                             uint32_t v, int lane) {
  const uint32_t w = sm[cbase + (int)(v >> 2) * 32 + lane];
  return (w >> ((v & 3) * 8)) & 0xffu;
}

__host__ __device__ inline int count_lut_stages(const StepArgs& a) {
  int n = 0;
  for (int s = 0; s < a.n_stages; ++s)
    if (a.stages[s].type == ST_LUT || a.stages[s].type == ST_EQ) ++n;
  return n;
}

// Stage this image's LUTs into shared memory (replicated per lane so the 32
// lookups of a warp hit 32 distinct banks) and fetch per-stage params.
// Must be followed by __syncthreads().
__device__ __forceinline__ void load_stages(const StepArgs& a, int img, uint32_t* sm,
                                            StageCtx& x, int nthreads) {
  int li = 0;
  for (int s = 0; s < a.n_stages; ++s) {
    const Stage st = a.stages[s];
    x.sd[s].on = 0;
    x.sd[s].dh = x.sd[s].ds = x.sd[s].dv = 0.f;
    if (st.type == ST_LUT || st.type == ST_EQ) {
      const uint8_t* tab = st.type == ST_EQ
                               ? a.tab.eq_luts + (size_t)img * 768
                               : a.tab.luts + ((size_t)img * a.tab.n_luts + st.lut) * 768;
      const uint32_t* t32 = reinterpret_cast<const uint32_t*>(tab);
      uint32_t* dst = sm + li * kLutWords;
      for (int idx = threadIdx.x; idx < kLutWords; idx += nthreads) dst[idx] = __ldg(t32 + (idx >> 5));
      ++li;
    } else {
      x.sd[s].on = fired_of(a.tab, img, st.slot) ? 1 : 0;
      if (st.type == ST_HSV) {
        const double* q = prm_of(a.tab, img, st.slot);
        x.sd[s].dh = (float)q[0];
        x.sd[s].ds = (float)q[1];
        x.sd[s].dv = (float)q[2];
      }
    }
  }
  x.n_lut = li;
}

__device__ __forceinline__ void apply_stages(const StepArgs& a, const StageCtx& x,
                                             const uint32_t* sm, int lane, uint32_t& r,
                                             uint32_t& g, uint32_t& b) {
  int li = 0;
#pragma unroll 1
  for (int s = 0; s < a.n_stages; ++s) {
    const int t = a.stages[s].type;
    if (t == ST_LUT || t == ST_EQ) {
      const uint32_t* L = sm + li * kLutWords;
      r = lut_look(L, 0, r, lane);
      g = lut_look(L, 2048, g, lane);
      b = lut_look(L, 4096, b, lane);
      ++li;
    } else if (t == ST_HSV) {
      if (x.sd[s].on) hsv_shift_px(x.sd[s].dh, x.sd[s].ds, x.sd[s].dv, r, g, b);
    } else {
      if (x.sd[s].on) {
        const uint32_t y = gray_px(r, g, b);
        r = g = b = y;
      }
    }
  }
}

// Store one 16-pixel output block of a u8 row: vector stores when the block is
// fully inside [0, W) (the caller guarantees the block start is 16-byte
// aligned), byte stores otherwise.
template <int C>
__device__ __forceinline__ void store_block(uint8_t* drow, int xb, int W, const uint32_t* w) {
  uint8_t* dp = drow + (ptrdiff_t)xb * C;
  if (xb >= 0 && xb + 16 <= W) {
    uint4* d4 = reinterpret_cast<uint4*>(dp);
#pragma unroll
    for (int v = 0; v < C; ++v) __stcs(d4 + v, make_uint4(w[4 * v], w[4 * v + 1], w[4 * v + 2], w[4 * v + 3]));
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int x = xb + i;
      if (x >= 0 && x < W) {
#pragma unroll
        for (int c = 0; c < C; ++c) dp[C * i + c] = (uint8_t)byte_of(w, C * i + c);
      }
    }
  }
}

// Store 16 pixels (r,g,b in p[3*i..]) as Normalize fp32 NCHW (O12), the 3x256
// fp32 LUT built by K0 in fp64.
__device__ __forceinline__ void store_nchw(const StepArgs& a, int img, int y, int xb,
                                           const uint32_t* px, int W, int H) {
  const size_t plane = (size_t)H * W;
  float* base = a.nchw + (size_t)img * 3 * plane + (size_t)y * W;
  const float* nl = a.tab.norm_lut;
  const bool vec = (W % 4 == 0) && xb >= 0 && xb + 16 <= W && (xb % 4 == 0);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    float* row = base + c * plane;
    if (vec) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float4 f = make_float4(__ldg(nl + c * 256 + px[3 * (4 * q + 0) + c]),
                               __ldg(nl + c * 256 + px[3 * (4 * q + 1) + c]),
                               __ldg(nl + c * 256 + px[3 * (4 * q + 2) + c]),
                               __ldg(nl + c * 256 + px[3 * (4 * q + 3) + c]));
        __stcs(reinterpret_cast<float4*>(row + xb) + q, f);
      }
    } else {
      for (int i = 0; i < 16; ++i) {
        const int x = xb + i;
        if (x >= 0 && x < W) row[x] = __ldg(nl + c * 256 + px[3 * i + c]);
      }
    }
  }
}

}  // namespace alb
