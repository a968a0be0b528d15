// equalize.cu -- K8 Equalize (reading R15), histogram + LUT; the apply pass is
// the pointwise kernel with an ST_EQ stage.
//   hist: per unit (image, 96 KB byte chunk) a warp-privatised shared-memory
//         histogram (8 warps x 768 bins) fed from 16-byte vector loads, then
//         reduced and added to the image's global histogram.
//   lut:  one CTA per image; per channel an exclusive block scan gives the CDF,
//         c_min = count of the first non-empty bin, D = N - c_min and
//         LUT[v] = (2*255*max(cdf[v]-c_min,0) + D) / (2*D) in 64-bit integers
//         (identity when D == 0).
#include "kernels.cuh"

namespace alb {

constexpr int kEqThreads = 256;

__global__ void __launch_bounds__(kEqThreads) k_eq_hist(EqArgs a) {
  __shared__ uint32_t h[kEqThreads / 32][768];
  const int2 unit = a.units[blockIdx.x];
  const int img = unit.x;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (kEqThreads / 32) * 768; i += kEqThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const alb_image_desc sd = a.sdesc[img];
  const int W = sd.width, H = sd.height;
  uint32_t* hw = h[warp];
  const bool flat = a.unit_size > 0;  // plan: whole image one segment, unit = byte chunk
  const int rows = flat ? 1 : H;
  const int seg = flat ? H * W * 3 : W * 3;
  for (int r = 0; r < rows; ++r) {
    const uint8_t* src = a.src + sd.offset + (size_t)r * sd.pitch;
    int b0 = 0, b1 = seg;
    if (flat) {
      b0 = unit.y * a.unit_size;
      b1 = min(seg, b0 + a.unit_size);
    } else if (r != unit.y) {
      continue;
    }
    // aligned body [bA, bE) in 16-byte vectors
    int bA = b0 + (int)((16 - (((uintptr_t)src + b0) & 15)) & 15);
    if (bA > b1) bA = b1;
    const int bE = bA + ((b1 - bA) / 16) * 16;
    for (int b = b0 + threadIdx.x; b < bA; b += kEqThreads) atomicAdd(&hw[(b % 3) * 256 + src[b]], 1u);
    for (int b = bE + threadIdx.x; b < b1; b += kEqThreads) atomicAdd(&hw[(b % 3) * 256 + src[b]], 1u);
    const uint4* s4 = reinterpret_cast<const uint4*>(src + bA);
    const int nv = (bE - bA) / 16;
    // thread -> contiguous run of vectors; the lanes of a warp take runs
    // kEqThreads/32 apart, i.e. far-apart pixels of the segment, so their
    // (spatially correlated) bins rarely collide in one shared atomic
    for (int v = threadIdx.x; v < nv; v += kEqThreads) {
      const uint4 t = __ldg(s4 + v);
      const uint32_t w[4] = {t.x, t.y, t.z, t.w};
      const int ph = (bA + 16 * v) % 3;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        int c = ph + (j % 3);
        c = c >= 3 ? c - 3 : c;
        atomicAdd(&hw[c * 256 + ((w[j >> 2] >> ((j & 3) * 8)) & 0xffu)], 1u);
      }
    }
  }
  __syncthreads();
  uint32_t* gh = a.hist + (size_t)img * 768;
  for (int i = threadIdx.x; i < 768; i += kEqThreads) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < kEqThreads / 32; ++w) s += h[w][i];
    if (s) atomicAdd(gh + i, s);
  }
}

__global__ void __launch_bounds__(256) k_eq_lut(EqArgs a) {
  const int img = a.img0 + blockIdx.x;
  const int v = threadIdx.x;
  __shared__ uint32_t sc[256];
  __shared__ uint32_t s_cmin;
  __shared__ uint32_t s_first;
  const alb_image_desc sd = a.sdesc[img];
  const int64_t N = (int64_t)sd.width * sd.height;
  if (!fired_of(a.tab, img, a.slot)) {  // gate not fired: the op is the identity
    for (int c = 0; c < 3; ++c) a.lut[(size_t)img * 768 + c * 256 + v] = (uint8_t)v;
    return;
  }
  for (int c = 0; c < 3; ++c) {
    const uint32_t hv = a.hist[(size_t)img * 768 + c * 256 + v];
    if (v == 0) s_first = 256;
    sc[v] = hv;
    __syncthreads();
    if (hv > 0) atomicMin(&s_first, (uint32_t)v);
    // inclusive scan (Hillis-Steele)
    for (int off = 1; off < 256; off <<= 1) {
      const uint32_t t = v >= off ? sc[v - off] : 0u;
      __syncthreads();
      sc[v] += t;
      __syncthreads();
    }
    if (v == (int)s_first) s_cmin = hv;
    __syncthreads();
    const int64_t cmin = s_first < 256 ? (int64_t)s_cmin : 0;
    const int64_t D = N - cmin;
    int out;
    if (D == 0) {
      out = v;
    } else {
      int64_t num = (int64_t)sc[v] - cmin;
      if (num < 0) num = 0;
      out = (int)((2 * 255 * num + D) / (2 * D));
    }
    a.lut[(size_t)img * 768 + c * 256 + v] = (uint8_t)out;
    __syncthreads();
  }
}

// Whole-image variant (flat images, one CTA of 1024 threads per image): lane-
// private histograms hl[bin][lane] (96 KB), so the 32 atomics of one warp
// instruction always hit 32 different banks (the warp-private layout above
// lets equal-bank bins collide: ~4 shared wavefronts per atomic).  The 32
// lanes' counts are summed with a rotated read order (conflict-free) and
// stored: the CTA owns the image's whole histogram.
constexpr int kEqLThreads = 1024;
constexpr size_t kEqLSmem = 768 * 32 * sizeof(uint32_t);

__global__ void __launch_bounds__(kEqLThreads) k_eq_hist_lane(EqArgs a) {
  extern __shared__ uint32_t hl[];  // [768][32]
  const int img = a.units[blockIdx.x].x;
  const int tid = threadIdx.x, lane = tid & 31;
  for (int i = tid; i < 768 * 32; i += kEqLThreads) hl[i] = 0;
  __syncthreads();
  const alb_image_desc sd = a.sdesc[img];
  const uint8_t* src = a.src + sd.offset;
  const int n = sd.height * sd.width * 3;
  uint32_t* hw = hl + lane;
  const uint32_t hl_base = (uint32_t)__cvta_generic_to_shared(hl) + 4u * (uint32_t)lane;
  int bA = (int)((16 - ((uintptr_t)src & 15)) & 15);
  if (bA > n) bA = n;
  const int bE = bA + ((n - bA) / 16) * 16;
  for (int b = tid; b < bA; b += kEqLThreads) atomicAdd(&hw[((b % 3) * 256 + src[b]) * 32], 1u);
  for (int b = bE + tid; b < n; b += kEqLThreads) atomicAdd(&hw[((b % 3) * 256 + src[b]) * 32], 1u);
  const uint4* s4 = reinterpret_cast<const uint4*>(src + bA);
  const int nv = (bE - bA) / 16;
  // vector v starts on channel (bA + v) % 3 (16 = 1 mod 3): thread tid's k-th
  // vector of pass j on (bA + tid + k + 2 j) % 3; the three bin-table bases
  // (shared byte address of (channel c, value x, lane) = base_c + 128 x) are
  // renamed per k and rotated by two per pass
  static_assert(kEqLThreads % 3 == 1 && (2 * kEqLThreads) % 3 == 2, "histogram vector phases");
  const int p0 = (bA + tid) % 3;
  uint32_t hb[3] = {hl_base + (uint32_t)p0 * 32768u, hl_base + (uint32_t)(p0 == 2 ? 0 : p0 + 1) * 32768u,
                    hl_base + (uint32_t)(p0 == 0 ? 2 : p0 - 1) * 32768u};
  for (int v0 = tid; v0 < nv; v0 += 2 * kEqLThreads) {
    uint4 t[2];
#pragma unroll
    for (int k = 0; k < 2; ++k)
      if (v0 + k * kEqLThreads < nv) t[k] = __ldcs(s4 + v0 + k * kEqLThreads);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int v = v0 + k * kEqLThreads;
      if (v >= nv) break;
      const uint32_t w[4] = {t[k].x, t[k].y, t[k].z, t[k].w};
      // one byte extract (PRMT), one IMAD, one RED per byte
      const uint32_t b0 = hb[k % 3], b1 = hb[(k + 1) % 3], b2 = hb[(k + 2) % 3];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t cb = (j % 3 == 0) ? b0 : ((j % 3 == 1) ? b1 : b2);
        const uint32_t x = __byte_perm(w[j >> 2], 0u, 0x4440u + (uint32_t)(j & 3));
        asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(x * 128u + cb) : "memory");
      }
    }
    const uint32_t r0 = hb[0];  // next pass starts two channels later
    hb[0] = hb[2];
    hb[2] = hb[1];
    hb[1] = r0;
  }
  __syncthreads();
  for (int i = tid; i < 768; i += kEqLThreads) {
    uint32_t sum = 0;
#pragma unroll 8
    for (int l = 0; l < 32; ++l) sum += hl[i * 32 + ((l + i) & 31)];
    a.hist[(size_t)img * 768 + i] = sum;
  }
}

void launch_eq_hist(const EqArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  if (a.unit_size == -1) {  // flat images, one unit per image
    persistent_grid((const void*)k_eq_hist_lane, kEqLThreads, kEqLSmem, a.n_units);  // smem attribute
    k_eq_hist_lane<<<a.n_units, kEqLThreads, kEqLSmem, s>>>(a);
  } else {
    k_eq_hist<<<a.n_units, kEqThreads, 0, s>>>(a);
  }
}
void launch_eq_lut(const EqArgs& a, cudaStream_t s) {
  if (a.n > 0) k_eq_lut<<<a.n, 256, 0, s>>>(a);
}

}  // namespace alb
