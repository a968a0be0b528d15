// point.cu -- pointwise colour kernel (K1 LUT ops, K6 ShiftHSV, K7 Grayscale,
// Equalize apply, Normalize output).  DESIGN.md O8-O12.
//
// Work unit = (image, 48 KB byte chunk of the image's contiguous segment) in
// flat mode (pitch == width*3 on both sides), or (image, row) otherwise.  The
// grid is persistent: CTA b owns a contiguous range of units (image-major), so
// the per-image LUTs (built by K0 in fp64) are staged in shared memory --
// lane-replicated, conflict-free -- only when the image changes.
//
// LUT-only chains run byte-wise on lane-coalesced 16-byte vectors (the channel
// of byte j of vector v is (v + j) % 3 because the body starts on a pixel
// boundary and 16 = 1 mod 3); chains that mix channels (HSV, gray) or write
// fp32 NCHW run pixel-wise on 48-byte (16-pixel) groups, two groups in flight
// per thread.  Unaligned heads and tails, and buffers that are not 16-byte
// co-aligned, take a per-pixel path.
#include <algorithm>

#include "stages.cuh"

namespace alb {

constexpr int kThreads = 256;
#ifndef ALB_LUT_U
#define ALB_LUT_U 6  // measured: 6 > 4 (Brightness 0.321 -> 0.317 ms) > 8 (register-limited occupancy)
#endif
constexpr int kU = ALB_LUT_U;   // 16-byte vectors in flight per thread (LUT path)
constexpr int kG = 2;   // 48-byte groups in flight per thread (pixel path)

struct Seg {
  const uint8_t* src;
  uint8_t* dst;
  int b0, b1, bA, bE;
  size_t pidx0, plane;
  float* plane0;
};

__device__ __forceinline__ Seg make_seg(const StepArgs& a, int2 unit) {
  const int img = unit.x;
  const alb_image_desc sd = a.sdesc[img];
  const int W = sd.width, H = sd.height;
  Seg s;
  s.dst = nullptr;
  if (a.flat) {
    s.src = a.src + sd.offset;
    if (a.dst) s.dst = a.dst + a.ddesc[img].offset;
    s.b0 = unit.y * a.unit_size;
    s.b1 = min(H * W * 3, s.b0 + a.unit_size);
    s.pidx0 = 0;
  } else {
    s.src = a.src + sd.offset + (size_t)unit.y * sd.pitch;
    if (a.dst) {
      const alb_image_desc dd = a.ddesc[img];
      s.dst = a.dst + dd.offset + (size_t)unit.y * dd.pitch;
    }
    s.b0 = 0;
    s.b1 = W * 3;
    s.pidx0 = (size_t)unit.y * W;
  }
  s.plane = (size_t)H * W;
  s.plane0 = a.normalize ? a.nchw + (size_t)img * 3 * s.plane : nullptr;
  s.bA = s.bE = s.b1;
  if (a.vec_ok) {
    int o = s.b0 + (int)((16 - (((uintptr_t)s.src + s.b0) & 15)) & 15);
    while ((o % 3) != 0) o += 16;
    if (o < s.b1) {
      s.bA = o;
      s.bE = o + ((s.b1 - o) / 48) * 48;
    }
  }
  return s;
}

template <int kOne>
__device__ __forceinline__ void scalar_edges(const StepArgs& a, const Seg& s, const StageCtx& x,
                                             const uint32_t* sm, int lane) {
  const float* nl = a.tab.norm_lut;
  auto px = [&](int p) {
    uint32_t r = s.src[3 * p], g = s.src[3 * p + 1], b = s.src[3 * p + 2];
    apply_stages_t<kOne>(x, sm, lane, r, g, b);
    if (a.normalize) {
      s.plane0[s.pidx0 + p] = nl[r];
      s.plane0[s.plane + s.pidx0 + p] = nl[256 + g];
      s.plane0[2 * s.plane + s.pidx0 + p] = nl[512 + b];
    } else {
      s.dst[3 * p] = (uint8_t)r;
      s.dst[3 * p + 1] = (uint8_t)g;
      s.dst[3 * p + 2] = (uint8_t)b;
    }
  };
  for (int p = s.b0 / 3 + threadIdx.x; p < s.bA / 3; p += kThreads) px(p);
  for (int p = s.bE / 3 + threadIdx.x; p < s.b1 / 3; p += kThreads) px(p);
}

// LUT-only chain (kNL1: exactly one LUT stage).  Single-stage lookups of
// byte j of word w (channel table base B_c 8 KB aligned, lane-replicated
// words: entry v at word (v >> 2) * 32 + lane):
//   addr  = ((w >> (8j - 5)) & 0x1F80) | (B_c | 4 lane)       SHF + LOP3
//   word  = LDS(addr)
// then four looked-up words pack into the output word with PRMT selectors
// built from (w & 0x03030303) for all four bytes at once.
// x >> (32 - k) computed by the multiplier: hi32(x * 2^k)
__device__ __forceinline__ uint32_t mulhi_pow2(uint32_t x, int k) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(1u << k));
  return r;
}
// byte permute with a run-time selector whose nibbles are known to be
// 0..7 (no sign-replicate bit): PTX prmt directly, so the compiler does not
// mask the selector first as it must for __byte_perm
__device__ __forceinline__ uint32_t prmt_raw(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Self-sampling LUT step (StepArgs::self_sample; one LUT stage, the plan's
// only step): image img's gate + params drawn here by thread 0 (sample_core,
// as K0), the composed 3 x 256 LUT built by the CTA in fp64 with the same
// lut_entry as K0, then replicated per lane into the stage's shared table
// exactly as load_stages does from K0's global table.
struct SelfLut {
  double prm[kMaxOps * kMaxParams];
  int32_t dims[2 * (kMaxOps + 1)];
  uint8_t fired[kMaxOps];
  uint32_t lut[192];  // 768 bytes
};
__device__ __forceinline__ void self_lut(const StepArgs& a, int img, uint32_t* sm, const StageCtx& x, SelfLut& t) {
  if (threadIdx.x == 0) {
    const alb_image_desc sd = a.sdesc[img];
    sample_core(a.ops, a.tab.n_ops, a.seed, a.first_image + (uint32_t)img, sd.height, sd.width, t.prm, t.fired,
                t.dims);
  }
  __syncthreads();
  uint8_t* l8 = reinterpret_cast<uint8_t*>(t.lut);
  for (int e = threadIdx.x; e < 768; e += kThreads) {
    const int c = e >> 8;
    int v = e & 255;
    for (int k = a.lut_k0; k < a.lut_k1; ++k)
      if (t.fired[k]) v = lut_entry(a.ops[k].kind, t.prm + k * kMaxParams, c, v);
    l8[e] = (uint8_t)v;
  }
  __syncthreads();
  uint32_t* dst = sm + x.smb[0];
  for (int idx = threadIdx.x; idx < kLutWords; idx += kThreads) dst[idx] = t.lut[idx >> 5];
}

template <bool kNL1>
#ifndef ALB_LUT_MINB
#define ALB_LUT_MINB 4
#endif
__global__ void __launch_bounds__(kThreads, ALB_LUT_MINB) k_point_lut(StepArgs a) {
  extern __shared__ uint32_t sm_raw[];
  const int lane = threadIdx.x & 31;
  // 8 KB-aligned LUT base (the launch reserves 8 KB of slack)
  const uint32_t raw_addr = (uint32_t)__cvta_generic_to_shared(sm_raw);
  uint32_t* sm = sm_raw + (((8192u - (raw_addr & 8191u)) & 8191u) >> 2);
  const uint32_t lb = (uint32_t)__cvta_generic_to_shared(sm) | (4u * lane);
  StageCtx x;
  init_stages(a, x);
  int u0, u1;
  unit_range(a.n_units, u0, u1);
  int cur_img = -1;
  __shared__ SelfLut self_t;
  for (int u = u0; u < u1; ++u) {
    const int2 unit = a.units[u];
    if (unit.x != cur_img) {
      __syncthreads();
      if (kNL1 && a.self_sample) self_lut(a, unit.x, sm, x, self_t);
      else load_stages(a, unit.x, sm, x, kThreads);
      __syncthreads();
      cur_img = unit.x;
    }
    const Seg s = make_seg(a, unit);
    scalar_edges<kStagesGeneric>(a, s, x, sm, lane);
    if (s.bE <= s.bA) continue;
    const int nv = (s.bE - s.bA) / 16;
    const uint4* s4 = reinterpret_cast<const uint4*>(s.src + s.bA);
    uint4* d4 = reinterpret_cast<uint4*>(s.dst + s.bA);
    // vector v starts on channel v % 3 (16 = 1 mod 3); with kThreads = 1 and
    // kThreads * kU = 0 (mod 3), thread t's k-th vector of every pass starts
    // on channel (t + k) % 3: the three channel table bases are rotated at
    // compile time instead of recomputed per vector
    static_assert(kThreads % 3 == 1 && (kThreads * kU) % 3 == 0, "vector phases must repeat per pass");
    const int pt = threadIdx.x % 3;
    const uint32_t cbt[3] = {lb + (uint32_t)pt * 8192u, lb + (uint32_t)(pt == 2 ? 0 : pt + 1) * 8192u,
                             lb + (uint32_t)(pt == 0 ? 2 : pt - 1) * 8192u};
    for (int v0 = threadIdx.x; v0 < nv; v0 += kThreads * kU) {
      uint4 in[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const int v = v0 + k * kThreads;
        if (v < nv) in[k] = __ldcs(s4 + v);
      }
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const int v = v0 + k * kThreads;
        if (v < nv) {
          const int ph = v % 3;  // channel of byte j is (ph + j) % 3 (segment starts on a pixel)
          uint32_t w[4] = {in[k].x, in[k].y, in[k].z, in[k].w};
          if constexpr (kNL1) {
            const uint32_t c0 = cbt[k % 3], c1 = cbt[(k + 1) % 3], c2 = cbt[(k + 2) % 3];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t r[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int jj = q * 4 + j;
                const uint32_t cb = (jj % 3 == 0) ? c0 : ((jj % 3 == 1) ? c1 : c2);
                // right shifts as IMAD.HI (FMA pipe; this loop is ALU-pipe bound)
                const uint32_t t = j == 0 ? (w[q] << 5) : mulhi_pow2(w[q], 37 - 8 * j);
                const uint32_t addr = (t & 0x1F80u) | cb;
                asm("ld.shared.u32 %0, [%1];" : "=r"(r[j]) : "r"(addr));
              }
              // byte (v & 3) of each looked-up word: selector nibbles from w & 0x03030303
              // (PRMT reads only the low 16 selector bits, and the result's
              // upper two bytes are dropped by the final permute)
              const uint32_t xs = w[q] & 0x03030303u;
              const uint32_t y = xs | (xs >> 4) | 0x00400040u;  // byte k: (v_k & 3) | (4 + (v_{k+1} & 3)) << 4
              const uint32_t lo = prmt_raw(r[0], r[1], y);
              const uint32_t hi = prmt_raw(r[2], r[3], y >> 16);
              w[q] = __byte_perm(lo, hi, 0x5410u);
            }
          } else {
            const int cb0 = ph * 2048;
            const int cb1 = (ph == 2 ? 0 : ph + 1) * 2048;
            const int cb2 = (ph == 0 ? 2 : ph - 1) * 2048;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t o = 0;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int jj = q * 4 + j;
                const int cb = (jj % 3 == 0) ? cb0 : ((jj % 3 == 1) ? cb1 : cb2);
                uint32_t val = (w[q] >> (8 * j)) & 0xffu;
                for (int t = 0; t < x.n_lut; ++t) val = lut_look(sm + t * kLutWords, cb, val, lane);
                o |= val << (8 * j);
              }
              w[q] = o;
            }
          }
          __stcs(d4 + v, make_uint4(w[0], w[1], w[2], w[3]));
        }
      }
    }
  }
}

// pixel-wise chain (HSV / gray / mixed / Normalize output); kNorm is
// compile-time so the unused output path is not issued per pixel
template <int kOne, bool kNorm>
#ifndef ALB_PX_MINB
#define ALB_PX_MINB 4
#endif
__global__ void __launch_bounds__(kThreads, ALB_PX_MINB) k_point_px(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31;
  StageCtx x;
  init_stages(a, x);
  int u0, u1;
  unit_range(a.n_units, u0, u1);
  int cur_img = -1;
  const float* nl = a.tab.norm_lut;
  __shared__ SelfLut self_t;  // self-sampling (HSV / gray only): thread 0's draws for the image
  for (int u = u0; u < u1; ++u) {
    const int2 unit = a.units[u];
    if (unit.x != cur_img) {
      __syncthreads();
      if (a.self_sample) {
        if (threadIdx.x == 0) {
          const alb_image_desc sd = a.sdesc[unit.x];
          sample_core(a.ops, a.tab.n_ops, a.seed, a.first_image + (uint32_t)unit.x, sd.height, sd.width, self_t.prm,
                      self_t.fired, self_t.dims);
        }
        __syncthreads();
        Tables t = a.tab;
        t.params = self_t.prm;
        t.fired = self_t.fired;
        load_px_params(a, t, 0, x);
      } else {
        load_stages(a, unit.x, sm, x, kThreads);
      }
      __syncthreads();
      cur_img = unit.x;
    }
    const Seg s = make_seg(a, unit);
    scalar_edges<kOne>(a, s, x, sm, lane);
    if (s.bE <= s.bA) continue;
    const int ng = (s.bE - s.bA) / 48;
    for (int g0 = threadIdx.x; g0 < ng; g0 += kThreads * kG) {
      uint32_t w[kG][12];
#pragma unroll
      for (int k = 0; k < kG; ++k) {
        const int gi = g0 + k * kThreads;
        if (gi < ng) {
          const uint4* s4 = reinterpret_cast<const uint4*>(s.src + s.bA + 48 * gi);
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const uint4 t = __ldcs(s4 + q);
            w[k][4 * q] = t.x; w[k][4 * q + 1] = t.y; w[k][4 * q + 2] = t.z; w[k][4 * q + 3] = t.w;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < kG; ++k) {
        const int gi = g0 + k * kThreads;
        if (gi >= ng) break;
        uint32_t o[12];
#pragma unroll
        for (int q = 0; q < 12; ++q) o[q] = 0;
        const size_t p0 = s.pidx0 + (s.bA + 48 * gi) / 3;
        if constexpr (kOne == ST_HSV && !kNorm) {  // pixel pairs on the paired fp32 pipe
          if (x.on[0]) {
            // 4 pixels (12 bytes = 3 words) at a time: each channel byte
            // becomes a biased float with one byte permute, and the 12
            // biased results pack into 3 words with 3 byte permutes each
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              uint32_t res[12];
#pragma unroll
              for (int pp = 0; pp < 4; pp += 2) {
                float2 Rb, Gb, Bb;
                auto bf = [&](int j) {  // byte j of the group -> 2^23 + byte
                  return __uint_as_float(__byte_perm(w[k][j >> 2], 0x4B000000u, 0x7540u | (uint32_t)(j & 3)));
                };
                const int j0 = 3 * (i + pp), j1 = j0 + 3;
                Rb = make_float2(bf(j0), bf(j1));
                Gb = make_float2(bf(j0 + 1), bf(j1 + 1));
                Bb = make_float2(bf(j0 + 2), bf(j1 + 2));
                uint32_t ro[2], go[2], bo[2];
                hsv_shift_px2b(x.dh[0], x.ds[0], x.dv[0], Rb, Gb, Bb, ro, go, bo);
                res[3 * pp] = ro[0]; res[3 * pp + 1] = go[0]; res[3 * pp + 2] = bo[0];
                res[3 * pp + 3] = ro[1]; res[3 * pp + 4] = go[1]; res[3 * pp + 5] = bo[1];
              }
#pragma unroll
              for (int m = 0; m < 3; ++m) {
                const uint32_t lo = __byte_perm(res[4 * m], res[4 * m + 1], 0x0040u);
                const uint32_t hi = __byte_perm(res[4 * m + 2], res[4 * m + 3], 0x0040u);
                o[(3 * i) / 4 + m] = __byte_perm(lo, hi, 0x5410u);
              }
            }
          } else {
#pragma unroll
            for (int q = 0; q < 12; ++q) o[q] = w[k][q];
          }
        } else
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint32_t px = rgbx_of(w[k], i);
          uint32_t r = px & 0xff, g = (px >> 8) & 0xff, b = px >> 16;
          apply_stages_t<kOne>(x, sm, lane, r, g, b);
          if constexpr (kNorm) {
            s.plane0[p0 + i] = nl[r];
            s.plane0[s.plane + p0 + i] = nl[256 + g];
            s.plane0[2 * s.plane + p0 + i] = nl[512 + b];
          } else {
            o[(3 * i) >> 2] |= r << (((3 * i) & 3) * 8);
            o[(3 * i + 1) >> 2] |= g << (((3 * i + 1) & 3) * 8);
            o[(3 * i + 2) >> 2] |= b << (((3 * i + 2) & 3) * 8);
          }
        }
        if constexpr (!kNorm) {
          uint4* d4 = reinterpret_cast<uint4*>(s.dst + s.bA + 48 * gi);
#pragma unroll
          for (int q = 0; q < 3; ++q)
            __stcs(d4 + q, make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]));
        }
      }
    }
  }
}

template <bool kNL1>
static void launch_lut(const StepArgs& a, size_t smem, cudaStream_t s) {
  smem += 8192;  // slack to align the LUT base to 8 KB
  persistent_grid((const void*)k_point_lut<kNL1>, kThreads, smem, a.n_units);  // smem attribute
  const int grid = a.n_units;  // one CTA per unit (whole images in flat mode)
  k_point_lut<kNL1><<<grid, kThreads, smem, s>>>(a);
}

template <int kOne, bool kNorm>
static void launch_px_n(const StepArgs& a, size_t smem, cudaStream_t s) {
  // without LUT stages there is no per-image shared state worth keeping:
  // one CTA per unit lets the hardware balance the ragged tail
  const int grid = smem == 0 ? a.n_units
                             : persistent_grid((const void*)k_point_px<kOne, kNorm>, kThreads, smem, a.n_units);
  k_point_px<kOne, kNorm><<<grid, kThreads, smem, s>>>(a);
}

template <int kOne>
static void launch_px(const StepArgs& a, size_t smem, cudaStream_t s) {
  if (a.normalize) launch_px_n<kOne, true>(a, smem, s);
  else launch_px_n<kOne, false>(a, smem, s);
}

// ============================================== single-pass Equalize (K8)
// Equalize then nothing else in the pointwise step, packed image rows, 16-byte
// co-aligned buffers: ONE kernel, one CTA of 1024 threads per image.
//   1. histogram: lane-private shared histograms hl[bin][lane] (conflict-free
//      atomics, as k_eq_hist_lane), 16-byte loads that keep their lines in
//      L2 (evict_last): the image is read from HBM once;
//   2. per channel: the 256 counts are scanned (warp shuffles), c_min is the
//      count of the first non-empty bin and LUT[v] = floor((2*255*max(cdf -
//      c_min, 0) + D) / (2 D)), D = N - c_min, in 64-bit integers (identity
//      when D == 0) -- the arithmetic of k_eq_lut / reading R15;
//   3. the LUT is replicated per lane over the histogram's shared memory and
//      the image is re-read (from L2, evict_first: last use) and written
//      through the single-LUT byte path of k_point_lut.
#ifndef ALB_EQF_THREADS
#define ALB_EQF_THREADS 1024  // one CTA per SM (measured: 1024 x 1 beats 512 x 2, 0.49 vs 0.56 ms)
#endif
constexpr int kEqF = ALB_EQF_THREADS;
#ifndef ALB_EQF_AHEAD
#define ALB_EQF_AHEAD 64  // images ahead the LUT pass prefetches into L2 (measured 16: 0.474, 37: 0.464, 56-74: 0.457, 100: 0.471, 148: 0.514, none: 0.469 ms)
#endif
constexpr int kEqPrefetchAhead = ALB_EQF_AHEAD;
constexpr size_t kEqFSmem = 8192 + 768 * 32 * 4 + 2 * 768 * 4 + 768;  // 8 KB alignment slack + hist + counts + prefixes + LUT

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ld_evict_last(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}

__global__ void __launch_bounds__(kEqF, 1024 / kEqF) k_eq_fused(StepArgs a) {
  extern __shared__ uint32_t sm_raw[];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t raw_addr = (uint32_t)__cvta_generic_to_shared(sm_raw);
  uint32_t* hl = sm_raw + (((8192u - (raw_addr & 8191u)) & 8191u) >> 2);  // 8 KB aligned, [768][32]
  uint32_t* cnt = hl + 768 * 32;                                          // [768]
  uint32_t* pre = cnt + 768;                                              // [768]
  uint8_t* lut8 = reinterpret_cast<uint8_t*>(pre + 768);                  // [768]
  __shared__ uint32_t wsum[24];
  __shared__ int first[3];
  const int img = a.img0 + blockIdx.x;  // one CTA per image of the launch range
  const alb_image_desc sd = a.sdesc[img];
  const uint8_t* src = a.src + sd.offset;
  const int n = sd.height * sd.width * 3;
  // gate not fired (a.stages[0] is this step's ST_EQ stage): identity LUT, no histogram
  const bool on = fired_of(a.tab, img, a.stages[0].slot);
  for (int i = tid; i < 768 * 32; i += kEqF) hl[i] = 0;
  if (tid < 3) first[tid] = 256;
  __syncthreads();
  // ---- 1. histogram
  if (on) {
    uint32_t* hw = hl + lane;
    const uint32_t hl_base = (uint32_t)__cvta_generic_to_shared(hl) + 4u * (uint32_t)lane;
    int bA = (int)((16 - ((uintptr_t)src & 15)) & 15);
    if (bA > n) bA = n;
    const int bE = bA + ((n - bA) / 16) * 16;
    for (int b = tid; b < bA; b += kEqF) atomicAdd(&hw[((b % 3) * 256 + src[b]) * 32], 1u);
    for (int b = bE + tid; b < n; b += kEqF) atomicAdd(&hw[((b % 3) * 256 + src[b]) * 32], 1u);
    const uint4* s4 = reinterpret_cast<const uint4*>(src + bA);
    const int nv = (bE - bA) / 16;
    constexpr int kV = 4;  // vectors in flight per thread (64 KB per SM)
    const uint64_t pol = policy_evict_last();
    // vector v starts on channel (bA + v) % 3; thread tid's k-th vector of
    // pass j on (bA + tid + k + j) % 3 (kEqF = 1 and kV * kEqF = 1 mod 3):
    // three bin-table bases, rotated by one per pass and renamed per k
    static_assert(kEqF % 3 == 1 && (kV * kEqF) % 3 == 1, "histogram vector phases");
    const int p0 = (bA + tid) % 3;
    uint32_t hb[3] = {hl_base + (uint32_t)p0 * 32768u, hl_base + (uint32_t)(p0 == 2 ? 0 : p0 + 1) * 32768u,
                      hl_base + (uint32_t)(p0 == 0 ? 2 : p0 - 1) * 32768u};
    for (int v0 = tid; v0 < nv; v0 += kV * kEqF) {
      uint4 t[kV];
#pragma unroll
      for (int k = 0; k < kV; ++k)
        if (v0 + k * kEqF < nv) t[k] = ld_evict_last(s4 + v0 + k * kEqF, pol);
#pragma unroll
      for (int k = 0; k < kV; ++k) {
        const int v = v0 + k * kEqF;
        if (v >= nv) break;
        const uint32_t w[4] = {t[k].x, t[k].y, t[k].z, t[k].w};
        const uint32_t b0 = hb[k % 3], b1 = hb[(k + 1) % 3], b2 = hb[(k + 2) % 3];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const uint32_t cb = (j % 3 == 0) ? b0 : ((j % 3 == 1) ? b1 : b2);
          const uint32_t xb = __byte_perm(w[j >> 2], 0u, 0x4440u + (uint32_t)(j & 3));
          asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(xb * 128u + cb) : "memory");
        }
      }
      const uint32_t r0 = hb[0];  // next pass starts one channel later
      hb[0] = hb[1];
      hb[1] = hb[2];
      hb[2] = r0;
    }
  }
  __syncthreads();
  // ---- 2. counts, per-channel inclusive scan, c_min, LUT (bin t = 0..767:
  //         channel c = t >> 8, value t & 255; the CTA's warps cover the bins in rounds)
  for (int t = tid; t < 768; t += kEqF) {
    uint32_t h = 0;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) h += hl[t * 32 + ((l + t) & 31)];
    uint32_t inc = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[t >> 5] = inc;
    if (h > 0) atomicMin(&first[t >> 8], t & 255);
    cnt[t] = h;
    pre[t] = inc;  // inclusive prefix within the bin's warp-sized group
  }
  __syncthreads();
  for (int t = tid; t < 768; t += kEqF) {
    const int c = t >> 8, v = t & 255;
    uint32_t inc = pre[t];
    for (int w = c * 8; w < (t >> 5); ++w) inc += wsum[w];  // earlier groups of the channel
    const int64_t N = (int64_t)sd.width * sd.height;
    const int64_t cmin = first[c] < 256 ? (int64_t)cnt[c * 256 + first[c]] : 0;
    const int64_t D = N - cmin;
    int out;
    if (D == 0) {
      out = v;
    } else {
      int64_t num = (int64_t)inc - cmin;
      if (num < 0) num = 0;
      out = (int)((2 * 255 * num + D) / (2 * D));
    }
    lut8[t] = on ? (uint8_t)out : (uint8_t)v;
  }
  __syncthreads();
  // ---- 3. lane-replicated LUT over the histogram, then the LUT pass
#ifndef ALB_EQF_NO_PREFETCH
  // an image kEqPrefetchAhead on (a CTA that starts while this wave drains)
  // is pulled into L2 by bulk prefetches while this CTA streams its LUT pass,
  // so that CTA's histogram pass reads L2 instead of waiting on HBM
  if (tid == 0) {
    const int nimg = img + kEqPrefetchAhead;
    if (nimg < a.n_img) {
      const alb_image_desc nd = a.sdesc[nimg];
      const uintptr_t p0 = (uintptr_t)(a.src + nd.offset) & ~(uintptr_t)15;
      const uintptr_t p1 = ((uintptr_t)(a.src + nd.offset) + (size_t)nd.height * nd.pitch + 15) & ~(uintptr_t)15;
      for (uintptr_t p = p0; p < p1; p += 65536) {
        const uint32_t sz = (uint32_t)min((uintptr_t)65536, p1 - p);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(sz) : "memory");
      }
    }
  }
#endif
  {
    const uint32_t* t32 = reinterpret_cast<const uint32_t*>(lut8);
    for (int idx = tid; idx < kLutWords; idx += kEqF) hl[idx] = t32[idx >> 5];
  }
  __syncthreads();
  uint32_t* sm = hl;
  StageCtx x;
  init_stages(a, x);  // one ST_EQ stage at shared word 0
  StepArgs ai = a;
  ai.unit_size = n;  // the whole image is one segment
  const Seg sg = make_seg(ai, make_int2(img, 0));
  if (tid < kThreads) scalar_edges<kStagesGeneric>(ai, sg, x, sm, lane);
  if (sg.bE <= sg.bA) return;
  const uint32_t lb = (uint32_t)__cvta_generic_to_shared(sm) | (4u * lane);
  const int nv = (sg.bE - sg.bA) / 16;
  const uint4* s4 = reinterpret_cast<const uint4*>(sg.src + sg.bA);
  uint4* d4 = reinterpret_cast<uint4*>(sg.dst + sg.bA);
  // channel table bases rotated at compile time (as k_point_lut)
  static_assert(kEqF % 3 == 1 && (kEqF * kU) % 3 == 0, "vector phases must repeat per pass");
  const int pt = tid % 3;
  const uint32_t cbt[3] = {lb + (uint32_t)pt * 8192u, lb + (uint32_t)(pt == 2 ? 0 : pt + 1) * 8192u,
                           lb + (uint32_t)(pt == 0 ? 2 : pt - 1) * 8192u};
  for (int v0 = tid; v0 < nv; v0 += kEqF * kU) {
    uint4 in[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int v = v0 + k * kEqF;
      if (v < nv) in[k] = __ldcs(s4 + v);
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int v = v0 + k * kEqF;
      if (v < nv) {
        uint32_t w[4] = {in[k].x, in[k].y, in[k].z, in[k].w};
        const uint32_t c0 = cbt[k % 3], c1 = cbt[(k + 1) % 3], c2 = cbt[(k + 2) % 3];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint32_t r[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int jj = q * 4 + j;
            const uint32_t cb = (jj % 3 == 0) ? c0 : ((jj % 3 == 1) ? c1 : c2);
            const uint32_t t = j == 0 ? (w[q] << 5) : mulhi_pow2(w[q], 37 - 8 * j);
            const uint32_t addr = (t & 0x1F80u) | cb;
            asm("ld.shared.u32 %0, [%1];" : "=r"(r[j]) : "r"(addr));
          }
          const uint32_t xs = w[q] & 0x03030303u;
          const uint32_t y = xs | (xs >> 4) | 0x00400040u;
          const uint32_t lo = prmt_raw(r[0], r[1], y);
          const uint32_t hi = prmt_raw(r[2], r[3], y >> 16);
          w[q] = __byte_perm(lo, hi, 0x5410u);
        }
        __stcs(d4 + v, make_uint4(w[0], w[1], w[2], w[3]));
      }
    }
  }
}

void launch_eq_fused(const StepArgs& a, cudaStream_t s) {
  const int n = a.n_img - a.img0;
  if (n <= 0) return;
  persistent_grid((const void*)k_eq_fused, kEqF, kEqFSmem, n);  // smem attribute
  k_eq_fused<<<n, kEqF, kEqFSmem, s>>>(a);
}

void launch_point(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  const int nl = count_lut_stages(a);
  const bool pure = !a.normalize && nl == a.n_stages && nl > 0;
  const size_t smem = (size_t)nl * kLutWords * 4;
  if (pure && nl == 1) {
    launch_lut<true>(a, smem, s);
  } else if (pure) {
    launch_lut<false>(a, smem, s);
  } else {
    const int mode = stage_mode(a);
    ALB_DISPATCH_STAGES(mode, launch_px, a, smem, s)
  }
}

}  // namespace alb
