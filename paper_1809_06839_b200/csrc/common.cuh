// common.cuh -- device helpers shared by the sm_100a kernels of the hot path.
// (No code is shared with oracle/; the formulas are re-derived from DESIGN.md.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/alb_b200.h"

namespace alb {

constexpr int kMaxOps = ALB_MAX_OPS;
constexpr int kMaxParams = ALB_MAX_PARAMS;
constexpr int kMaxStages = 4;   // pointwise stages fused into one kernel
constexpr int kMaxLuts = 8;     // LUT stages per pipeline

// ---------------------------------------------------------------- O1 Philox
// Philox4x32-10 (Salmon et al. SC'11).  Counter (image, slot, block, tag=0),
// key (seed lo, seed hi); draw j uses block j>>1, words 2(j&1), 2(j&1)+1.
__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

__host__ __device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  return c;
}

// exact 53-bit double in [0,1): ((a>>5)*2^26 + (b>>6)) * 2^-53
__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
  return __dmul_rn(__dadd_rn(__dmul_rn((double)(a >> 5), 67108864.0), (double)(b >> 6)),
                   1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double draw_u(uint64_t seed, uint32_t img, int slot, int j) {
  const uint4 o = philox10(make_uint4(img, (uint32_t)slot, (uint32_t)(j >> 1), 0u),
                           make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  return (j & 1) ? u53(o.z, o.w) : u53(o.x, o.y);
}

// lo + (hi - lo) * u, no contraction
__device__ __forceinline__ double urange(double lo, double hi, double u) {
  return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
}

// floor(u * n), clamped to n - 1
__device__ __forceinline__ int uint_draw(double u, int n) {
  int k = (int)floor(__dmul_rn(u, (double)n));
  return k > n - 1 ? n - 1 : k;
}

// round half up + clamp to [0,255], in double
__device__ __forceinline__ int clip_round_d(double v) {
  double r = floor(__dadd_rn(v, 0.5));
  r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
  return (int)r;
}

__host__ __device__ __forceinline__ int reflect101(int i, int n) {
  if (n == 1) return 0;
  const int period = 2 * n - 2;
  int k = i < 0 ? -i : i;
  k = k % period;
  return k >= n ? period - k : k;
}

__host__ __device__ __forceinline__ bool is_lut_kind(int k) {
  return k == ALB_BRIGHTNESS || k == ALB_CONTRAST || k == ALB_BRIGHTNESS_CONTRAST ||
         k == ALB_GAMMA || k == ALB_SHIFT_RGB;
}

// ------------------------------------------------------- pointwise stages
enum StageType : int32_t { ST_LUT = 0, ST_HSV = 1, ST_GRAY = 2, ST_EQ = 3 };

struct Stage {
  int32_t type;
  int32_t slot;   // op slot (HSV/GRAY: gate + params)
  int32_t lut;    // LUT table index (ST_LUT)
  int32_t pad;
};

// per-apply tables in the workspace
struct Tables {
  const double* params;   // [n][n_ops][8]
  const uint8_t* fired;   // [n][n_ops]
  const int32_t* dims;    // [n][n_ops+1][2] (h, w) each slot sees
  const uint8_t* luts;    // [n][n_luts][768]
  const float* norm_lut;  // [3][256]
  const uint8_t* eq_luts; // [n][768] (Equalize, R15)
  int32_t n_ops;
  int32_t n_luts;
  const double* grid;     // [n][n_grid][kGridStride] GridDistortion knot displacements
  int32_t n_grid;
};

// GridDistortion knot tables: e^x[0..n] at +0, e^y[0..n] at +kGridAxis (reading R31)
constexpr int kGridAxis = ALB_GRID_MAX_STEPS + 1;
constexpr int kGridStride = 2 * kGridAxis;

__device__ __forceinline__ const double* prm_of(const Tables& t, int img, int slot) {
  return t.params + ((size_t)img * t.n_ops + slot) * kMaxParams;
}
__device__ __forceinline__ bool fired_of(const Tables& t, int img, int slot) {
  return t.fired[(size_t)img * t.n_ops + slot] != 0;
}

// ---- paired fp32 helpers (sm_100 f32x2 pipe)
__device__ __forceinline__ unsigned long long f2u(float2 v) {
  return ((unsigned long long)__float_as_uint(v.y) << 32) | __float_as_uint(v.x);
}
__device__ __forceinline__ float2 u2f(unsigned long long u) {
  return make_float2(__uint_as_float((uint32_t)u), __uint_as_float((uint32_t)(u >> 32)));
}
// round-toward-minus-infinity paired add: floor(v) + 1.5*2^23 for |v| < 2^22
__device__ __forceinline__ float2 fadd2_rm(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(r);
}

// ---------------------------------------------------------------- HSV (fp32)
// hexcone RGB->HSV, shift (h mod 360, s/v clamped), HSV->RGB, round half up
// (O9, reading R29).  Branch-free (no lane divergence):
//  * bytes -> floats as 2^23 + byte (one LOP each); max/min/differences are
//    exact in that biased form;
//  * hue in sixths, dominant channel with ties r > g > b:
//      h6 = num / d + off + dh6w,  dh6w = (dh / 60) mod 6 in [0, 6)
//    (per image), so h6 in [-1, 11); d = 0 gives num = 0, off = 0;
//    reciprocals are clamped to 2 so 0 * rcp(0) = 0 (d, mx are integers);
//  * channel n (5, 3, 1 for R, G, B): k = h6 + n in [0, 16) and
//      c = v - v s sat(2 - min(|k-2|, |k-8|, |k-14|)),
//    the periodic form of SPEC.md:419's sector table sat(min(k', 4-k')),
//    k' = k mod 6; h6 is moved down one period when >= 5 (exactly), which
//    leaves h6 in [-1, 5), k < 10, so the |k-14| term is never the minimum;
//    for R |k-2| >= 2 and for B |k-8| > 2, so only G needs two terms;
//  * out = floor(255 c + 0.5) from the mantissa of a round-down add.
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void hsv_shift_px(float dh6w, float ds, float dv, uint32_t& r, uint32_t& g,
                                             uint32_t& b) {
  const float M = 8388608.f;  // 2^23
  const float Rb = __uint_as_float(r | 0x4B000000u), Gb = __uint_as_float(g | 0x4B000000u),
              Bb = __uint_as_float(b | 0x4B000000u);
  const float mxb = fmaxf(Rb, fmaxf(Gb, Bb));
  const float mnb = fminf(Rb, fminf(Gb, Bb));
  const float d = mxb - mnb;
  const float mx = mxb - M;
  const bool isr = mxb == Rb;
  const bool isg = !isr && mxb == Gb;
  const float pa = isr ? Gb : (isg ? Bb : Rb);
  const float pb = isr ? Bb : (isg ? Rb : Gb);
  const float off = isr ? dh6w : (isg ? dh6w + 2.f : dh6w + 4.f);
  const float h6r = fmaf(pa - pb, fminf(rcp_approx(d), 2.f), off);  // in [-1, 11)
  // one period down when h6 >= 5 (exact: Sterbenz), so k = h6 + n < 10 and the
  // |k - 14| term can never be the minimum: fl(h6 - 6 + c) == fl(h6 + (c - 6))
  const float h6 = h6r >= 5.f ? h6r - 6.f : h6r;
  const float s = __saturatef(fmaf(d, fminf(rcp_approx(mx), 2.f), ds));
  const float v = __saturatef(fmaf(mx, 1.f / 255.f, dv));
  const float vs = v * s;
  // channel n: k = h6 + n, t = sat(2 - min(|k - 2|, |k - 8|)).  With h6 in
  // [-1, 5): for R (n = 5) |k - 2| = h6 + 3 >= 2, for B (n = 1) |k - 8| =
  // 7 - h6 > 2, so those terms can only give t = 0 -- the same value the
  // other term gives there (exact; verified on every byte triple by the GPU
  // parity tests) -- and R, B need one term each; G needs both.
  auto out = [&](float t) {
    const float y = fmaf(255.f, fmaf(-vs, t, v), 0.5f);
    return __float_as_uint(__fadd_rd(y, M)) & 0xffu;
  };
  r = out(__saturatef(2.f - fabsf(h6 + (5.f - 8.f))));
  g = out(__saturatef(2.f - fminf(fabsf(h6 + (3.f - 2.f)), fabsf(h6 + (3.f - 8.f)))));
  b = out(__saturatef(2.f - fabsf(h6 + (1.f - 2.f))));
}

// Two pixels at once on the paired fp32 pipe (FADD2 / FFMA2 / FMUL2 where
// both pixels run the same operation; min / max / select / reciprocal per
// pixel).  Every per-pixel value equals hsv_shift_px's bit for bit (a paired
// op rounds each lane exactly like its scalar op), so the fused resample /
// affine paths (scalar) and the pointwise kernel (paired) agree.
__device__ __forceinline__ float2 f2add(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
// Core on biased floats (2^23 + byte) in, biased bit patterns out (byte in
// bits 0-7, 0x4B0000 above): callers that unpack / pack with byte permutes
// skip the per-channel masks and ORs.
// the part after the hue (shared by both hsv_shift_px2b variants)
__device__ __forceinline__ void hsv_tail2(float ds, float dv, float2 d, float2 mx, float2 rm, float2 h6r,
                                          uint32_t (&ro)[2], uint32_t (&go)[2], uint32_t (&bo)[2]) {
  const float M = 8388608.f;
  const float2 h6 = make_float2(h6r.x >= 5.f ? h6r.x - 6.f : h6r.x, h6r.y >= 5.f ? h6r.y - 6.f : h6r.y);
  float2 sv = f2fma(d, rm, make_float2(ds, ds));
  sv = make_float2(__saturatef(sv.x), __saturatef(sv.y));
  float2 vv = f2fma(mx, make_float2(1.f / 255.f, 1.f / 255.f), make_float2(dv, dv));
  vv = make_float2(__saturatef(vv.x), __saturatef(vv.y));
  const float2 vs = __fmul2_rn(vv, sv);
  const float2 nvs = make_float2(-vs.x, -vs.y);
  // t per channel as hsv_shift_px (R and B need one term each, G both)
  auto emit = [&](float2 t, uint32_t (&out)[2]) {
    const float2 y = f2fma(make_float2(255.f, 255.f), f2fma(nvs, t, vv), make_float2(0.5f, 0.5f));
    const float2 q = fadd2_rm(y, make_float2(M, M));  // both pixels' round-down adds in one op
    out[0] = __float_as_uint(q.x);
    out[1] = __float_as_uint(q.y);
  };
  const float2 kr = f2add(h6, make_float2(5.f - 8.f, 5.f - 8.f));
  emit(make_float2(__saturatef(2.f - fabsf(kr.x)), __saturatef(2.f - fabsf(kr.y))), ro);
  const float2 kg2 = f2add(h6, make_float2(3.f - 2.f, 3.f - 2.f));
  const float2 kg8 = f2add(h6, make_float2(3.f - 8.f, 3.f - 8.f));
  emit(make_float2(__saturatef(2.f - fminf(fabsf(kg2.x), fabsf(kg8.x))),
                   __saturatef(2.f - fminf(fabsf(kg2.y), fabsf(kg8.y)))), go);
  const float2 kb = f2add(h6, make_float2(1.f - 2.f, 1.f - 2.f));
  emit(make_float2(__saturatef(2.f - fabsf(kb.x)), __saturatef(2.f - fabsf(kb.y))), bo);
}
// kCand3: the hue of both pixels from three candidates (dominant R, G, B)
// computed on the paired pipe -- differences exact on biased integers, the
// same fma a selected operand pair gives, so bit-identical -- then two
// selects per pixel instead of six (ShiftHSV 0.475 -> 0.470 ms, cfg4 fused
// resampler 0.308 -> 0.307 ms, A/B); -DALB_HSV_SEL_PAIRS: the operand selects.
template <bool kCand3 = true>
__device__ __forceinline__ void hsv_shift_px2b(float dh6w, float ds, float dv, float2 Rb, float2 Gb, float2 Bb,
                                               uint32_t (&ro)[2], uint32_t (&go)[2], uint32_t (&bo)[2]) {
  const float M = 8388608.f;
#ifdef ALB_HSV_SEL_PAIRS
  constexpr bool kC3 = false;
#else
  constexpr bool kC3 = kCand3;
#endif
  if constexpr (kC3) {
    float2 mxb, mnb;
    bool isr[2], isg[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float R = i ? Rb.y : Rb.x, G = i ? Gb.y : Gb.x, B = i ? Bb.y : Bb.x;
      const float hi = fmaxf(R, fmaxf(G, B)), lo = fminf(R, fminf(G, B));
      isr[i] = hi == R;
      isg[i] = !isr[i] && hi == G;
      if (i) { mxb.y = hi; mnb.y = lo; }
      else { mxb.x = hi; mnb.x = lo; }
    }
    const float2 d = f2add(mxb, make_float2(-mnb.x, -mnb.y));
    const float2 mx = f2add(mxb, make_float2(-M, -M));
    const float2 rd = make_float2(fminf(rcp_approx(d.x), 2.f), fminf(rcp_approx(d.y), 2.f));
    const float2 rm = make_float2(fminf(rcp_approx(mx.x), 2.f), fminf(rcp_approx(mx.y), 2.f));
    const float2 hr = f2fma(f2add(Gb, make_float2(-Bb.x, -Bb.y)), rd, make_float2(dh6w, dh6w));
    const float2 hg = f2fma(f2add(Bb, make_float2(-Rb.x, -Rb.y)), rd, make_float2(dh6w + 2.f, dh6w + 2.f));
    const float2 hb = f2fma(f2add(Rb, make_float2(-Gb.x, -Gb.y)), rd, make_float2(dh6w + 4.f, dh6w + 4.f));
    const float2 h6r = make_float2(isr[0] ? hr.x : (isg[0] ? hg.x : hb.x), isr[1] ? hr.y : (isg[1] ? hg.y : hb.y));
    hsv_tail2(ds, dv, d, mx, rm, h6r, ro, go, bo);
  } else {
    float2 mxb, mnb, pa, pb, off;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float R = i ? Rb.y : Rb.x, G = i ? Gb.y : Gb.x, B = i ? Bb.y : Bb.x;
      const float hi = fmaxf(R, fmaxf(G, B)), lo = fminf(R, fminf(G, B));
      const bool isr = hi == R;
      const bool isg = !isr && hi == G;
      const float A_ = isr ? G : (isg ? B : R), B_ = isr ? B : (isg ? R : G);
      const float o = isr ? dh6w : (isg ? dh6w + 2.f : dh6w + 4.f);
      if (i) { mxb.y = hi; mnb.y = lo; pa.y = A_; pb.y = B_; off.y = o; }
      else { mxb.x = hi; mnb.x = lo; pa.x = A_; pb.x = B_; off.x = o; }
    }
    const float2 d = f2add(mxb, make_float2(-mnb.x, -mnb.y));
    const float2 mx = f2add(mxb, make_float2(-M, -M));
    const float2 rd = make_float2(fminf(rcp_approx(d.x), 2.f), fminf(rcp_approx(d.y), 2.f));
    const float2 rm = make_float2(fminf(rcp_approx(mx.x), 2.f), fminf(rcp_approx(mx.y), 2.f));
    const float2 h6r = f2fma(f2add(pa, make_float2(-pb.x, -pb.y)), rd, off);
    hsv_tail2(ds, dv, d, mx, rm, h6r, ro, go, bo);
  }
}
__device__ __forceinline__ void hsv_shift_px2(float dh6w, float ds, float dv, uint32_t (&r)[2], uint32_t (&g)[2],
                                              uint32_t (&b)[2]) {
  float2 Rb, Gb, Bb;
  Rb.x = __uint_as_float(r[0] | 0x4B000000u); Rb.y = __uint_as_float(r[1] | 0x4B000000u);
  Gb.x = __uint_as_float(g[0] | 0x4B000000u); Gb.y = __uint_as_float(g[1] | 0x4B000000u);
  Bb.x = __uint_as_float(b[0] | 0x4B000000u); Bb.y = __uint_as_float(b[1] | 0x4B000000u);
  uint32_t ro[2], go[2], bo[2];
  hsv_shift_px2b(dh6w, ds, dv, Rb, Gb, Bb, ro, go, bo);
  r[0] = ro[0] & 0xffu; r[1] = ro[1] & 0xffu; g[0] = go[0] & 0xffu; g[1] = go[1] & 0xffu;
  b[0] = bo[0] & 0xffu; b[1] = bo[1] & 0xffu;
}

// exact BT.601 luma (299R + 587G + 114B + 500) / 1000
__device__ __forceinline__ uint32_t gray_px(uint32_t r, uint32_t g, uint32_t b) {
  return (299u * r + 587u * g + 114u * b + 500u) / 1000u;
}

// ------------------------------------------------------------- byte windows
// Load NW words = bytes [p, p + 4*NW) at arbitrary alignment using 16-byte
// aligned vector loads; only vectors intersecting [lo, hi) are read (the rest
// stay zero), so reads never leave the 16-byte blocks of valid data.
template <int NW>
__device__ __forceinline__ void load_window(const uint8_t* __restrict__ p, const uint8_t* lo,
                                            const uint8_t* hi, uint32_t (&w)[NW]) {
  constexpr int NV = (NW + 4 + 3) / 4;
  const uintptr_t a = (uintptr_t)p;
  const uint8_t* base = (const uint8_t*)(a & ~(uintptr_t)15);
  const int sh = (int)(a & 15);
  uint32_t r[NV * 4];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const uint8_t* q = base + 16 * v;
    uint4 x = make_uint4(0, 0, 0, 0);
    if (q < hi && q + 16 > lo) x = __ldg(reinterpret_cast<const uint4*>(q));
    r[4 * v + 0] = x.x; r[4 * v + 1] = x.y; r[4 * v + 2] = x.z; r[4 * v + 3] = x.w;
  }
  const int qw = sh >> 2, kb = (sh & 3) * 8;
  uint32_t t1[NV * 4 - 1];
#pragma unroll
  for (int i = 0; i < NV * 4 - 1; ++i) t1[i] = (qw & 1) ? r[i + 1] : r[i];
  uint32_t t2[NW + 1];
#pragma unroll
  for (int i = 0; i < NW + 1; ++i) t2[i] = (qw & 2) ? t1[i + 2] : t1[i];
#pragma unroll
  for (int i = 0; i < NW; ++i) w[i] = __funnelshift_r(t2[i], t2[i + 1], kb);
}

// 256-bit streaming global accesses (sm_100: LDG/STG.E.EF.ENL2.256), 32-byte aligned
__device__ __forceinline__ void ld256_cs(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.cs.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void ld256_nc(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void st256_cs(void* p, const uint32_t (&r)[8]) {
  asm volatile("st.global.cs.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]),
               "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

__device__ __forceinline__ uint32_t byte_of(const uint32_t* w, int j) {
  return (w[j >> 2] >> ((j & 3) * 8)) & 0xffu;
}

// First offset a0 in [0, 16*C) with (addr + a0) % 16 == 0 and a0 % C == 0.
template <int C>
__device__ __forceinline__ int first_aligned_px_offset(uintptr_t addr) {
  int a0 = (int)((16 - (addr & 15)) & 15);
  if (C == 3) {
    while (a0 % 3) a0 += 16;
  }
  return a0;
}

__device__ __forceinline__ int ld_desc_h(const alb_image_desc* d) { return d->height; }

}  // namespace alb
