// stages.cuh -- pointwise stage chain (LUT / Equalize LUT / HSV / gray) shared
// by the pointwise, resample and affine kernels so fused and unfused paths
// execute the same arithmetic.  At most kMaxStages stages per kernel; the
// chain is unrolled so per-stage state lives in registers.
#pragma once
#include "kernels.cuh"

namespace alb {

constexpr int kLutWords = 3 * 64 * 32;  // one lane-replicated LUT stage (24 KB)

struct StageCtx {
  int type[kMaxStages];
  int on[kMaxStages];
  int smb[kMaxStages];  // shared-memory word offset of the stage's LUT
  float dh[kMaxStages], ds[kMaxStages], dv[kMaxStages];
  int n;
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

// Static part of the context (types, LUT slots) -- no memory traffic.
__device__ __forceinline__ void init_stages(const StepArgs& a, StageCtx& x) {
  x.n = a.n_stages;
  int li = 0;
#pragma unroll
  for (int s = 0; s < kMaxStages; ++s) {
    x.type[s] = s < a.n_stages ? a.stages[s].type : -1;
    x.on[s] = 0;
    x.dh[s] = x.ds[s] = x.dv[s] = 0.f;
    x.smb[s] = li * kLutWords;
    if (x.type[s] == ST_LUT || x.type[s] == ST_EQ) ++li;
  }
  x.n_lut = li;
}

// Stage image `img`'s LUTs into shared memory (replicated per lane so a
// warp's 32 lookups hit 32 distinct banks) and fetch per-stage params.
// Caller brackets with __syncthreads().
__device__ __forceinline__ void load_stages(const StepArgs& a, int img, uint32_t* sm, StageCtx& x,
                                            int nthreads);

// Per-stage HSV / gray params of image `img` of table view `tab` (no LUT stages).
__device__ __forceinline__ void load_px_params(const StepArgs& a, const Tables& tab, int img, StageCtx& x) {
#pragma unroll
  for (int s = 0; s < kMaxStages; ++s) {
    const int t = x.type[s];
    if (t == ST_HSV || t == ST_GRAY) {
      x.on[s] = fired_of(tab, img, a.stages[s].slot) ? 1 : 0;
      if (t == ST_HSV) {
        const double* q = prm_of(tab, img, a.stages[s].slot);
        double w = q[0] / 60.0;          // hue shift in sixths of a turn, wrapped to [0, 6)
        w -= 6.0 * floor(w / 6.0);
        x.dh[s] = (float)w;
        x.ds[s] = (float)q[1];
        x.dv[s] = (float)q[2];
      }
    }
  }
}

__device__ __forceinline__ void load_stages(const StepArgs& a, int img, uint32_t* sm, StageCtx& x,
                                            int nthreads) {
#pragma unroll
  for (int s = 0; s < kMaxStages; ++s) {
    const int t = x.type[s];
    if (t == ST_LUT || t == ST_EQ) {
      const uint8_t* tab = t == ST_EQ
                               ? a.tab.eq_luts + (size_t)img * 768
                               : a.tab.luts + ((size_t)img * a.tab.n_luts + a.stages[s].lut) * 768;
      const uint32_t* t32 = reinterpret_cast<const uint32_t*>(tab);
      uint32_t* dst = sm + x.smb[s];
      for (int idx = threadIdx.x; idx < kLutWords; idx += nthreads) dst[idx] = __ldg(t32 + (idx >> 5));
    } else if (t == ST_HSV || t == ST_GRAY) {
      x.on[s] = fired_of(a.tab, img, a.stages[s].slot) ? 1 : 0;
      if (t == ST_HSV) {
        const double* q = prm_of(a.tab, img, a.stages[s].slot);
        double w = q[0] / 60.0;          // hue shift in sixths of a turn, wrapped to [0, 6)
        w -= 6.0 * floor(w / 6.0);
        x.dh[s] = (float)w;
        x.ds[s] = (float)q[1];
        x.dv[s] = (float)q[2];
      }
    }
  }
}

__device__ __forceinline__ void apply_stages(const StageCtx& x, const uint32_t* sm, int lane,
                                             uint32_t& r, uint32_t& g, uint32_t& b) {
#pragma unroll
  for (int s = 0; s < kMaxStages; ++s) {
    const int t = x.type[s];
    if (t == ST_LUT || t == ST_EQ) {
      const uint32_t* L = sm + x.smb[s];
      r = lut_look(L, 0, r, lane);
      g = lut_look(L, 2048, g, lane);
      b = lut_look(L, 4096, b, lane);
    } else if (t == ST_HSV) {
      if (x.on[s]) hsv_shift_px(x.dh[s], x.ds[s], x.dv[s], r, g, b);
    } else if (t == ST_GRAY) {
      if (x.on[s]) {
        const uint32_t y = gray_px(r, g, b);
        r = g = b = y;
      }
    }
  }
}

// Compile-time stage program: kOne = -2 no stages, -1 generic chain, the
// type of the single stage (its LUT, if any, sits at shared word 0), or one of
// the two-stage programs HSV -> LUT (cfg4's ShiftHSV -> BrightnessContrast) and
// LUT -> HSV (the single LUT sits at shared word 0 in both).
constexpr int kStagesNone = -2, kStagesGeneric = -1, kStagesHsvLut = 10, kStagesLutHsv = 11;

template <int kOne>
__device__ __forceinline__ void apply_stages_t(const StageCtx& x, const uint32_t* sm, int lane,
                                               uint32_t& r, uint32_t& g, uint32_t& b) {
  if constexpr (kOne == kStagesNone) {
    return;
  } else if constexpr (kOne == ST_LUT || kOne == ST_EQ) {
    r = lut_look(sm, 0, r, lane);
    g = lut_look(sm, 2048, g, lane);
    b = lut_look(sm, 4096, b, lane);
  } else if constexpr (kOne == ST_HSV) {
    if (x.on[0]) hsv_shift_px(x.dh[0], x.ds[0], x.dv[0], r, g, b);
  } else if constexpr (kOne == ST_GRAY) {
    if (x.on[0]) {
      const uint32_t y = gray_px(r, g, b);
      r = g = b = y;
    }
  } else if constexpr (kOne == kStagesHsvLut) {
    if (x.on[0]) hsv_shift_px(x.dh[0], x.ds[0], x.dv[0], r, g, b);
    r = lut_look(sm, 0, r, lane);
    g = lut_look(sm, 2048, g, lane);
    b = lut_look(sm, 4096, b, lane);
  } else if constexpr (kOne == kStagesLutHsv) {
    r = lut_look(sm, 0, r, lane);
    g = lut_look(sm, 2048, g, lane);
    b = lut_look(sm, 4096, b, lane);
    if (x.on[1]) hsv_shift_px(x.dh[1], x.ds[1], x.dv[1], r, g, b);
  } else {
    apply_stages(x, sm, lane, r, g, b);
  }
}

// Two pixels through the stage program (kOne as apply_stages_t): HSV runs on
// the paired fp32 pipe (hsv_shift_px2, bit-identical per pixel), LUT / gray
// stages per pixel.
template <int kOne>
__device__ __forceinline__ void apply_stages2_t(const StageCtx& x, const uint32_t* sm, int lane,
                                                uint32_t (&r)[2], uint32_t (&g)[2], uint32_t (&b)[2]) {
  if constexpr (kOne == kStagesNone) {
    return;
  } else if constexpr (kOne == ST_HSV) {
    if (x.on[0]) hsv_shift_px2(x.dh[0], x.ds[0], x.dv[0], r, g, b);
  } else if constexpr (kOne == kStagesHsvLut) {
    if (x.on[0]) hsv_shift_px2(x.dh[0], x.ds[0], x.dv[0], r, g, b);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      r[h] = lut_look(sm, 0, r[h], lane);
      g[h] = lut_look(sm, 2048, g[h], lane);
      b[h] = lut_look(sm, 4096, b[h], lane);
    }
  } else if constexpr (kOne == kStagesLutHsv) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      r[h] = lut_look(sm, 0, r[h], lane);
      g[h] = lut_look(sm, 2048, g[h], lane);
      b[h] = lut_look(sm, 4096, b[h], lane);
    }
    if (x.on[1]) hsv_shift_px2(x.dh[1], x.ds[1], x.dv[1], r, g, b);
  } else if constexpr (kOne == kStagesGeneric) {
#pragma unroll
    for (int s = 0; s < kMaxStages; ++s) {
      const int t = x.type[s];
      if (t == ST_LUT || t == ST_EQ) {
        const uint32_t* L = sm + x.smb[s];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          r[h] = lut_look(L, 0, r[h], lane);
          g[h] = lut_look(L, 2048, g[h], lane);
          b[h] = lut_look(L, 4096, b[h], lane);
        }
      } else if (t == ST_HSV) {
        if (x.on[s]) hsv_shift_px2(x.dh[s], x.ds[s], x.dv[s], r, g, b);
      } else if (t == ST_GRAY) {
        if (x.on[s]) {
#pragma unroll
          for (int h = 0; h < 2; ++h) r[h] = g[h] = b[h] = gray_px(r[h], g[h], b[h]);
        }
      }
    }
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h) apply_stages_t<kOne>(x, sm, lane, r[h], g[h], b[h]);
  }
}

inline int stage_mode(const StepArgs& a) {
  if (a.n_stages == 0) return kStagesNone;
  if (a.n_stages == 1) return a.stages[0].type;
  if (a.n_stages == 2) {
    const int t0 = a.stages[0].type, t1 = a.stages[1].type;
    const bool l0 = t0 == ST_LUT || t0 == ST_EQ, l1 = t1 == ST_LUT || t1 == ST_EQ;
    if (t0 == ST_HSV && l1) return kStagesHsvLut;
    if (l0 && t1 == ST_HSV) return kStagesLutHsv;
  }
  return kStagesGeneric;
}

// Launch helper: instantiate kernel template K<mode> for the step's stage program.
#define ALB_DISPATCH_STAGES(mode, KERNEL, ...)                 \
  switch (mode) {                                               \
    case kStagesNone: KERNEL<kStagesNone>(__VA_ARGS__); break;  \
    case ST_LUT: KERNEL<ST_LUT>(__VA_ARGS__); break;            \
    case ST_EQ: KERNEL<ST_EQ>(__VA_ARGS__); break;              \
    case ST_HSV: KERNEL<ST_HSV>(__VA_ARGS__); break;            \
    case ST_GRAY: KERNEL<ST_GRAY>(__VA_ARGS__); break;          \
    case kStagesHsvLut: KERNEL<kStagesHsvLut>(__VA_ARGS__); break; \
    case kStagesLutHsv: KERNEL<kStagesLutHsv>(__VA_ARGS__); break; \
    default: KERNEL<kStagesGeneric>(__VA_ARGS__); break;        \
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

// Store 16 pixels (r,g,b in px[3*i..]) as Normalize fp32 NCHW (O12), the 3x256
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

// Warp-cooperative store of a row segment: lane l holds pixel l (R | G<<8 |
// B<<16); pixels l < nvalid are written to base[3l .. 3l+2].  The 3*nvalid
// bytes are regrouped with two shuffles + one byte permute per lane into
// 4-byte-aligned words (coalesced STG.32); only the partial first/last words
// fall back to byte stores.  All 32 lanes must call it.
__device__ __forceinline__ void warp_store_rgb(uint8_t* base, int nvalid, uint32_t px, int lane) {
  const int off = (int)((uintptr_t)base & 3);
  uint8_t* wb = base - off;
  const int k0 = 4 * lane - off;             // first segment byte of word `lane`
  const int qa = k0 >= 0 ? k0 / 3 : -1;      // pixel holding byte k0
  const int r = k0 - 3 * qa;                 // 0..2
  const uint32_t pa = __shfl_sync(0xffffffffu, px, qa < 0 ? 0 : qa);
  const uint32_t pb = __shfl_sync(0xffffffffu, px, qa + 1 > 31 ? 31 : qa + 1);
  const uint32_t sel = r == 0 ? 0x4210u : (r == 1 ? 0x5421u : 0x6542u);
  const uint32_t w = __byte_perm(pa, pb, sel);
  const int nbytes = 3 * nvalid;
  if (k0 >= 0 && k0 + 4 <= nbytes) {
    *reinterpret_cast<uint32_t*>(wb + 4 * lane) = w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k0 + j;
      if (k >= 0 && k < nbytes) wb[4 * lane + j] = (uint8_t)(w >> (8 * j));
    }
  }
  // words beyond lane 31 (segment of 32 px spans up to 25 words: never)
}

// Warp-cooperative copy of n bytes from a 16-byte-aligned shared buffer to a
// global address of any alignment: 16-byte aligned STG.128 for the body
// (source realigned from two LDS.128 with a funnel shift), byte stores for the
// unaligned head/tail.  Caller brackets with __syncwarp().
__device__ __forceinline__ void warp_copy_row(uint8_t* dst, const uint8_t* src, int n, int lane) {
  const int head = min(n, (int)((16 - ((uintptr_t)dst & 15)) & 15));
  if (lane < head) dst[lane] = src[lane];
  const int nb = (n - head) >> 4;
  const int sh = head & 15;  // source misalignment of every body block
  const int qw = sh >> 2, kb = (sh & 3) * 8;
  for (int k = lane; k < nb; k += 32) {
    const int so = head + 16 * k;
    const uint4* p = reinterpret_cast<const uint4*>(src + (so & ~15));
    const uint4 v0 = p[0];
    uint4 v1 = make_uint4(0, 0, 0, 0);
    if (sh) v1 = p[1];
    const uint32_t r[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    uint32_t t1[7], w[5];
#pragma unroll
    for (int i = 0; i < 7; ++i) t1[i] = (qw & 1) ? r[i + 1] : r[i];
#pragma unroll
    for (int i = 0; i < 5; ++i) w[i] = (qw & 2) ? t1[i + 2] : t1[i];
    uint4 o;
    o.x = __funnelshift_r(w[0], w[1], kb);
    o.y = __funnelshift_r(w[1], w[2], kb);
    o.z = __funnelshift_r(w[2], w[3], kb);
    o.w = __funnelshift_r(w[3], w[4], kb);
    __stcs(reinterpret_cast<uint4*>(dst + so), o);
  }
  const int t0 = head + 16 * nb;
  for (int b = t0 + lane; b < n; b += 32) dst[b] = src[b];
}

// CTA-cooperative copy of `rows` rows of n bytes from shared memory (row
// pitch spitch, 16-byte aligned) to global rows of any alignment: per row one
// item per aligned 16-byte block plus one item each for the unaligned head
// and tail bytes.
// x / d for 0 <= x < 2^20 via a precomputed magic (magic_of(d) == 0 means d == 1)
__host__ __device__ __forceinline__ uint32_t magic_of(uint32_t d) {
  return d <= 1 ? 0u : 0xffffffffu / d + 1u;
}__device__ __forceinline__ int fdiv(int x, uint32_t m) {
  return m == 0 ? x : (int)__umulhi((uint32_t)x, m);
}

// magic = magic_of((n >> 4) + 2), precomputed by the caller (one thread)
__device__ __forceinline__ void cta_copy_rows(uint8_t* dst0, int dpitch, const uint8_t* src0,
                                              int spitch, int rows, int n, int nthreads,
                                              uint32_t magic) {
  const int npr = (n >> 4) + 2;
  for (int it = threadIdx.x; it < rows * npr; it += nthreads) {
    const int r = fdiv(it, magic);
    const int k = it - r * npr;
    uint8_t* dst = dst0 + (size_t)r * dpitch;
    const uint8_t* src = src0 + r * spitch;
    const int head = min(n, (int)((16 - ((uintptr_t)dst & 15)) & 15));
    const int nb = (n - head) >> 4;
    if (k < nb) {
      const int so = head + 16 * k;
      const int sh = head & 15, qw = sh >> 2, kb = (sh & 3) * 8;
      const uint4* p = reinterpret_cast<const uint4*>(src + (so & ~15));
      const uint4 v0 = p[0];
      const uint4 v1 = sh ? p[1] : make_uint4(0, 0, 0, 0);
      const uint32_t q[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
      uint32_t t1[7], w[5];
#pragma unroll
      for (int i = 0; i < 7; ++i) t1[i] = (qw & 1) ? q[i + 1] : q[i];
#pragma unroll
      for (int i = 0; i < 5; ++i) w[i] = (qw & 2) ? t1[i + 2] : t1[i];
      __stcs(reinterpret_cast<uint4*>(dst + so),
             make_uint4(__funnelshift_r(w[0], w[1], kb), __funnelshift_r(w[1], w[2], kb),
                        __funnelshift_r(w[2], w[3], kb), __funnelshift_r(w[3], w[4], kb)));
    } else if (k == nb) {
      for (int b = 0; b < head; ++b) dst[b] = src[b];
    } else if (k == nb + 1) {
      for (int b = head + 16 * nb; b < n; ++b) dst[b] = src[b];
    }
  }
}

// Pixel i (0..15) of a 48-byte window as an RGBx word (one byte permute).
__device__ __forceinline__ uint32_t rgbx_of(const uint32_t (&w)[12], int i) {
  const int q = (3 * i) >> 2, k = (3 * i) & 3;
  const uint32_t hi = w[q + 1 < 12 ? q + 1 : 11];
  return __byte_perm(w[q], hi, (uint32_t)k * 0x111u + 0x210u) & 0xffffffu;
}

// Pixel i (0..15) of a 48-byte window as an RGBx word, byte 3 unspecified.
__device__ __forceinline__ uint32_t rgbx_raw(const uint32_t (&w)[12], int i) {
  const int q = (3 * i) >> 2, k = (3 * i) & 3;
  const uint32_t hi = w[q + 1 < 12 ? q + 1 : 11];
  return __byte_perm(w[q], hi, (uint32_t)k * 0x111u + 0x210u);
}

// Bilinear blend of 4 RGBx taps (O5/O7 weights), fp32, per channel
//   h0 = fma(fx, p10 - p00, p00 + .5); h1 = fma(fx, p11 - p01, p01 + .5);
//   v  = fma(fy, h1 - h0, h0);   out = floor(v)        (= round_half_up)
// Bytes become floats via the 2^23 magic (byte permute); channel pairs run
// on the paired fp32 pipe.  Returns the three rounded channels as the bit
// patterns of floor(v) + 2^23 (byte in bits 0-7).
__device__ __forceinline__ void bilerp3(uint32_t t00, uint32_t t10, uint32_t t01, uint32_t t11,
                                        float2 f, uint32_t& r, uint32_t& g, uint32_t& b) {
  constexpr uint32_t kM = 0x4B000000u;  // 2^23
  auto cv = [](uint32_t t, uint32_t c) { return __uint_as_float(__byte_perm(t, kM, 0x7540u | c)); };
  const float2 P00 = make_float2(cv(t00, 0), cv(t00, 1)), P10 = make_float2(cv(t10, 0), cv(t10, 1));
  const float2 P01 = make_float2(cv(t01, 0), cv(t01, 1)), P11 = make_float2(cv(t11, 0), cv(t11, 1));
  const float2 B0 = make_float2(cv(t00, 2), cv(t01, 2)), B1 = make_float2(cv(t10, 2), cv(t11, 2));
  const float2 nMh = make_float2(-8388607.5f, -8388607.5f);  // -(2^23 - 0.5), exact
  const float2 fx2 = make_float2(f.x, f.x);
  const float2 H0 = __ffma2_rn(fx2, __fadd2_rn(P10, make_float2(-P00.x, -P00.y)), __fadd2_rn(P00, nMh));
  const float2 H1 = __ffma2_rn(fx2, __fadd2_rn(P11, make_float2(-P01.x, -P01.y)), __fadd2_rn(P01, nMh));
  const float2 HB = __ffma2_rn(fx2, __fadd2_rn(B1, make_float2(-B0.x, -B0.y)), __fadd2_rn(B0, nMh));
  const float2 V = __ffma2_rn(make_float2(f.y, f.y), __fadd2_rn(H1, make_float2(-H0.x, -H0.y)), H0);
  const float vb = fmaf(f.y, HB.y - HB.x, HB.x);
  const float2 R2 = fadd2_rm(V, make_float2(8388608.f, 8388608.f));
  r = __float_as_uint(R2.x);
  g = __float_as_uint(R2.y);
  b = __float_as_uint(__fadd_rd(vb, 8388608.f));
}

// bilerp3 on raw tap rows: u = bytes R0 G0 B0 R1 | G1 B1 . . of the upper
// tap row (the two pixels x0, x0 + 1), v likewise for the lower row.  The
// same arithmetic as bilerp3, bit for bit; only the byte selections differ.
__device__ __forceinline__ void bilerp3_raw(uint32_t u0, uint32_t u1, uint32_t v0, uint32_t v1, float2 f,
                                            uint32_t& r, uint32_t& g, uint32_t& b) {
  constexpr uint32_t kM = 0x4B000000u;  // 2^23
  auto cv = [](uint32_t t, uint32_t c) { return __uint_as_float(__byte_perm(t, kM, 0x7540u | c)); };
  const float2 P00 = make_float2(cv(u0, 0), cv(u0, 1)), P10 = make_float2(cv(u0, 3), cv(u1, 0));
  const float2 P01 = make_float2(cv(v0, 0), cv(v0, 1)), P11 = make_float2(cv(v0, 3), cv(v1, 0));
  const float2 B0 = make_float2(cv(u0, 2), cv(v0, 2)), B1 = make_float2(cv(u1, 1), cv(v1, 1));
  const float2 nMh = make_float2(-8388607.5f, -8388607.5f);
  const float2 fx2 = make_float2(f.x, f.x);
  const float2 H0 = __ffma2_rn(fx2, __fadd2_rn(P10, make_float2(-P00.x, -P00.y)), __fadd2_rn(P00, nMh));
  const float2 H1 = __ffma2_rn(fx2, __fadd2_rn(P11, make_float2(-P01.x, -P01.y)), __fadd2_rn(P01, nMh));
  const float2 HB = __ffma2_rn(fx2, __fadd2_rn(B1, make_float2(-B0.x, -B0.y)), __fadd2_rn(B0, nMh));
  const float2 V = __ffma2_rn(make_float2(f.y, f.y), __fadd2_rn(H1, make_float2(-H0.x, -H0.y)), H0);
  const float vb = fmaf(f.y, HB.y - HB.x, HB.x);
  const float2 R2 = fadd2_rm(V, make_float2(8388608.f, 8388608.f));
  r = __float_as_uint(R2.x);
  g = __float_as_uint(R2.y);
  b = __float_as_uint(__fadd_rd(vb, 8388608.f));
}

// Copy bytes [lo, hi) of one 16-byte chunk, smem -> global, both 16-aligned:
// naturally aligned pieces when the range touches an end of the chunk.
__device__ __forceinline__ void copy_partial(uint8_t* d, const uint8_t* s, int lo, int hi) {
  if (hi == 16) {
    int p = lo;
    if (p & 1) { d[p] = s[p]; p += 1; }
    if (p & 2) { *reinterpret_cast<uint16_t*>(d + p) = *reinterpret_cast<const uint16_t*>(s + p); p += 2; }
    if (p & 4) { *reinterpret_cast<uint32_t*>(d + p) = *reinterpret_cast<const uint32_t*>(s + p); p += 4; }
    if (p & 8) { *reinterpret_cast<uint2*>(d + p) = *reinterpret_cast<const uint2*>(s + p); }
  } else if (lo == 0) {
    int p = 0;
    if (hi & 8) { *reinterpret_cast<uint2*>(d) = *reinterpret_cast<const uint2*>(s); p = 8; }
    if (hi & 4) { *reinterpret_cast<uint32_t*>(d + p) = *reinterpret_cast<const uint32_t*>(s + p); p += 4; }
    if (hi & 2) { *reinterpret_cast<uint16_t*>(d + p) = *reinterpret_cast<const uint16_t*>(s + p); p += 2; }
    if (hi & 1) d[p] = s[p];
  } else {
    for (int b = lo; b < hi; ++b) d[b] = s[b];
  }
}

// CTA copy of `rows` buffered rows to global.  Row r's n bytes sit in the
// buffer at [r*pitch + phase, +n) where phase = (global row address) & 15, so
// every 16-byte chunk is aligned on both sides.  Full chunks first (kFull =
// max full chunks per row), then one item per partial head / tail chunk.
template <int kFull, int NT>
__device__ __forceinline__ void copy_rows_out(uint8_t* g0, int gpitch, const uint8_t* b0, int bpitch,
                                              int rows, int n) {
  for (int it = threadIdx.x; it < rows * kFull; it += NT) {
    const int r = it / kFull, k = it - r * kFull;
    uint8_t* grow = g0 + (size_t)r * gpitch;
    const int o = (int)((uintptr_t)grow & 15);
    const int c = ((o + 15) >> 4) + k;
    if (16 * c + 16 <= o + n)
      __stcs(reinterpret_cast<uint4*>(grow - o + 16 * c),
             *reinterpret_cast<const uint4*>(b0 + r * bpitch + 16 * c));
  }
  for (int it = threadIdx.x; it < 2 * rows; it += NT) {
    const bool head = it < rows;
    const int r = head ? it : it - rows;
    uint8_t* grow = g0 + (size_t)r * gpitch;
    const int o = (int)((uintptr_t)grow & 15);
    const uint8_t* s = b0 + r * bpitch;
    uint8_t* d = grow - o;
    const int e = o + n;
    if (head) {  // chunk 0 when the row does not start on a chunk boundary
      if (o > 0) copy_partial(d, s, o, min(e, 16));
    } else {     // last chunk when the row does not end on a chunk boundary
      const int c = e >> 4, hi = e & 15;
      if (hi > 0 && (c > 0 || o == 0)) copy_partial(d + 16 * c, s + 16 * c, 0, hi);
    }
  }
}

// Warp copy of one buffered row to global: the row's n bytes sit in `buf`
// (16-byte aligned) at [phase, phase + n), phase = (global row address) & 15,
// so every 16-byte chunk is aligned on both sides.
__device__ __forceinline__ void warp_copy_row_phased(uint8_t* grow, const uint8_t* buf, int n, int lane) {
  const int o = (int)((uintptr_t)grow & 15);
  uint8_t* d = grow - o;
  const int e = o + n;
  const int cf = (o + 15) >> 4, ce = e >> 4;
  for (int c = cf + lane; c < ce; c += 32)
    __stcs(reinterpret_cast<uint4*>(d + 16 * c), *reinterpret_cast<const uint4*>(buf + 16 * c));
  if (lane == 0 && o > 0) copy_partial(d, buf, o, min(e, 16));
  if (lane == 1) {
    const int hi = e & 15;
    if (hi > 0 && (ce > 0 || o == 0)) copy_partial(d + 16 * ce, buf + 16 * ce, 0, hi);
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar), "r"(parity) : "memory");
}

// TMA bulk copy global -> shared (16-byte aligned, size multiple of 16),
// completion counted on the mbarrier `bar`
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}

// Contiguous range of units for CTA b of G (persistent kernels): consecutive
// units belong mostly to the same image, so per-image state is reloaded only
// when the image changes.
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

__device__ __forceinline__ void unit_range(int n_units, int& u0, int& u1) {
  const long long G = gridDim.x, b = blockIdx.x;
  u0 = (int)(b * n_units / G);
  u1 = (int)((b + 1) * n_units / G);
}

}  // namespace alb
