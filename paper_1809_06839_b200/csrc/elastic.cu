// elastic.cu -- K12 ElasticTransform (reading
// R32): the displacement field is rebuilt on chip from the counter-based raw
// planes (nothing per-image in HBM), blurred in fp64 and used to remap the
// image (and mask) from global memory.
//
//   raw  u, v = -1 + 2 u53(draw j), j = 1 + y W + x  (u) / 1 + H W + y W + x  (v)
//   bx   = sum_k w_k raw[y][refl(x + k)]   (ascending k, acc = fma(w_k, v, acc))
//   d    = alpha * sum_k w_k bx[refl(y + k)][x]
//   out  = sample(x + dx, y + dy)          (bilinear / nearest, constant or reflect-101)
//
// The weights w_k are computed once per plan on the host (libm exp, the same
// bits the oracle computes) and the blur runs in fp64 in the definition's
// order, so source coordinates are bit-identical to the oracle's; only the
// bilinear blend runs in fp32 (bilerp3).
//
// Work unit = (image, strip of TW = 8U output columns, band of kElBand output
// rows); one CTA of 8 warps slides down the band in chunks of 32 rows:
//   produce: the next <= 32 halo rows, plane u then v: raw values (one Philox
//            block per pair of horizontally adjacent pixels) into a row buffer,
//            then the x pass with lane = halo row and warp = U output columns
//            (register-blocked: U accumulators, a rotating window of U weights,
//            one shared load per U FMAs) into a ring of 2r + 32 rows per plane;
//   consume: the y pass for 32 output rows, lane = column, U rows per thread
//            (same register blocking), dx and dy of a pixel in one thread, then
//            the remap of those pixels straight from registers.
// Weights are zero-padded so the unrolled loops need no bounds (a zero-weight
// term fma(0, v, acc) leaves acc unchanged).
#include "stages.cuh"

namespace alb {

constexpr int kElThreads = 256;
constexpr int kElWarps = 8;
constexpr int kElChunk = 32;  // rows per produce / consume step (= lanes)

// tap steps of a U-output register block: outputs i < U, taps k <= 2r, m = i + k,
// rounded up to a multiple of U
__host__ __device__ constexpr int el_msteps(int r, int U) { return (2 * r + U + U - 1) / U * U; }

// layout (doubles): padded weights | raw rows | ring u | ring v
struct ElLayout {
  int nw, rw, ring_rows, raw_off, ring_off;
  __host__ __device__ ElLayout(int r, int U) {
    const int M = el_msteps(r, U);
    nw = M + U;                               // padded weight table
    rw = (8 * U + M) | 1;                     // raw row stride (odd: conflict-free lane = row)
    ring_rows = 2 * r + kElChunk;
    raw_off = (nw + 1) & ~1;
    ring_off = raw_off + kElChunk * rw;
  }
  __host__ __device__ size_t bytes(int U) const {
    return ((size_t)ring_off + (size_t)2 * ring_rows * (8 * U + 1)) * 8;
  }
};

int elastic_strip(int r) { return r <= 24 ? 64 : 32; }

size_t elastic_smem(int r) {
  const int U = elastic_strip(r) / 8;
  return ElLayout(r, U).bytes(U);
}

// exact -1 + 2 u53(a, b) (O1): the 53-bit integer scaled by 2^-52, minus 1
__device__ __forceinline__ double raw_of(uint32_t a, uint32_t b) {
  const unsigned long long n = ((unsigned long long)(a >> 5) << 26) | (b >> 6);
  return __fma_rn((double)n, 1.0 / 4503599627370496.0, -1.0);
}

// reflect-101 with the in-range and single-reflection cases first
__device__ __forceinline__ int refl(int i, int n) {
  if ((unsigned)i < (unsigned)n) return i;
  if (n == 1) return 0;
  const int k = i < 0 ? -i : 2 * n - 2 - i;
  return (unsigned)k < (unsigned)n ? k : reflect101(i, n);
}

template <int U>
__global__ void __launch_bounds__(kElThreads) k_elastic(StepArgs a) {
  constexpr int TW = 8 * U;
  constexpr int RS = TW + 1;  // ring row stride: x-pass stores (lane = row) hit distinct banks
  extern __shared__ double esm[];
  const int r = a.g_r;
  const ElLayout L(r, U);
  const int M = el_msteps(r, U);      // tap steps per output block
  double* wz = esm;                   // wz[t] = w_{t - (U-1)}, zero outside [0, 2r]
  double* raw = esm + L.raw_off;      // [32][rw]
  double* ring = esm + L.ring_off;    // [2][ring_rows][RS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int2 unit = a.units[blockIdx.x];
  const int img = unit.x;
  const alb_image_desc sd = a.sdesc[img];
  const int W = sd.width, H = sd.height;
  const int x0 = (unit.y & 0xffff) * TW, yb0 = (unit.y >> 16) * kElBand;
  const int yb1 = min(H, yb0 + kElBand);
  const bool fired = fired_of(a.tab, img, a.slot0);
  const bool reflect = a.border == ALB_BORDER_REFLECT_101;
  const bool nearest = a.interp == ALB_INTERP_NEAREST;
  const uint8_t* simg = a.src + sd.offset;
  const alb_image_desc dd = a.ddesc[img];
  uint8_t* dimg = a.dst + dd.offset;
  const uint8_t* smk = a.mdst ? a.msrc + a.msdesc[img].offset : nullptr;
  const int mps = a.mdst ? a.msdesc[img].pitch : 0;
  uint8_t* dmk = a.mdst ? a.mdst + a.mddesc[img].offset : nullptr;
  const int mpd = a.mdst ? a.mddesc[img].pitch : 0;

  // sample output pixel (x, y) at (x + dx, y + dy) and store it
  auto remap = [&](int x, int y, double dxv, double dyv) {
    double xs = (double)x, ys = (double)y;
    if (fired) {
      xs = __dadd_rn(xs, dxv);
      ys = __dadd_rn(ys, dyv);
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
      bool i0, i1, j0, j1;
      const int px0 = border_idx(xa, W, reflect, i0), px1 = border_idx(xa + 1, W, reflect, i1);
      const int py0 = border_idx(ya, H, reflect, j0), py1 = border_idx(ya + 1, H, reflect, j1);
      const uint8_t* r0 = simg + (size_t)py0 * sd.pitch;
      const uint8_t* r1 = simg + (size_t)py1 * sd.pitch;
      const uint32_t t00 = (i0 && j0) ? fetch_rgb(r0, px0) : a.fill;
      const uint32_t t10 = (i1 && j0) ? fetch_rgb(r0, px1) : a.fill;
      const uint32_t t01 = (i0 && j1) ? fetch_rgb(r1, px0) : a.fill;
      const uint32_t t11 = (i1 && j1) ? fetch_rgb(r1, px1) : a.fill;
      uint32_t rr, gg, bb;
      bilerp3(t00, t10, t01, t11, f, rr, gg, bb);
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
  };

  if (!fired) {  // identity: the same sampler with a zero field
    for (int i = tid; i < (yb1 - yb0) * TW; i += kElThreads) {
      const int x = x0 + (i % TW), y = yb0 + i / TW;
      if (x < W) remap(x, y, 0.0, 0.0);
    }
    return;
  }

  for (int t = tid; t < L.nw; t += kElThreads) {
    const int k = t - (U - 1);
    wz[t] = (k >= 0 && k <= 2 * r) ? a.gauss[k] : 0.0;
  }
  const int RW = TW + 2 * r;  // raw columns a halo row needs
  const int RR = L.ring_rows;
  for (int i = tid; i < 2 * RR * RS; i += kElThreads) ring[i] = 0.0;  // rows past the data meet zero weights
  for (int i = tid; i < kElChunk * (L.rw - RW); i += kElThreads) {  // finite padding columns
    const int row = i / (L.rw - RW);
    raw[row * L.rw + RW + (i - row * (L.rw - RW))] = 0.0;
  }
  const uint32_t gi = a.first_image + (uint32_t)img;
  const uint2 key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32));
  const int plane_j = W * H;

  // produce halo rows [Y0, Y0 + n) (image coordinates before reflection), n <= 32
  auto produce = [&](int Y0, int n, int slot0) {
    for (int plane = 0; plane < 2; ++plane) {
      const int j0 = 1 + plane * plane_j;
      // raw values: warp = row, lane = pair of columns sharing one Philox block
      const int npair = (RW + 2) >> 1;
      for (int row = warp; row < n; row += kElWarps) {
        const int jr = j0 + refl(Y0 + row, H) * W;
        const int J0 = jr + (x0 - r);  // j of raw column 0 if unreflected
        double* dst = raw + row * L.rw;
        for (int p = lane; p < npair; p += 32) {
          const int q0 = 2 * p - (J0 & 1);
          const int xa = x0 - r + q0;
          if (xa >= 0 && xa + 1 < W) {  // both unreflected: one block
            const uint4 o = philox10(make_uint4(gi, (uint32_t)a.slot0, (uint32_t)((J0 + q0) >> 1), 0u), key);
            if (q0 >= 0) dst[q0] = raw_of(o.x, o.y);
            if (q0 + 1 < RW) dst[q0 + 1] = raw_of(o.z, o.w);
          } else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int q = q0 + e;
              if (q < 0 || q >= RW) continue;
              const int j = jr + refl(x0 - r + q, W);
              const uint4 o = philox10(make_uint4(gi, (uint32_t)a.slot0, (uint32_t)(j >> 1), 0u), key);
              dst[q] = (j & 1) ? raw_of(o.z, o.w) : raw_of(o.x, o.y);
            }
          }
        }
      }
      __syncthreads();
      // x pass: lane = halo row, warp = output columns [U warp, U warp + U)
      if (lane < n) {
        const double* src = raw + lane * L.rw + U * warp;
        double acc[U], wv[U];
#pragma unroll
        for (int i = 0; i < U; ++i) acc[i] = 0.0;
#pragma unroll
        for (int j = 0; j < U - 1; ++j) wv[j] = wz[j];
        for (int mb = 0; mb < M; mb += U) {
#pragma unroll
          for (int s = 0; s < U; ++s) {
            wv[(s + U - 1) % U] = wz[mb + s + U - 1];
            const double v = src[mb + s];
#pragma unroll
            for (int i = 0; i < U; ++i) acc[i] = __fma_rn(wv[(s + U - 1 - i) % U], v, acc[i]);
          }
        }
        int sl = slot0 + lane;
        if (sl >= RR) sl -= RR;
        double* d = ring + ((size_t)plane * RR + sl) * RS + U * warp;
#pragma unroll
        for (int i = 0; i < U; ++i) d[i] = acc[i];
      }
      __syncthreads();
    }
  };

  int produced = yb0 - r;  // next halo row to produce
  int pslot = 0;           // its ring slot
  for (int Q = yb0; Q < yb1; Q += kElChunk) {
    const int need = min(Q + kElChunk, yb1) - 1 + r;  // last halo row this chunk reads
    while (produced <= need) {
      const int n = min(kElChunk, need - produced + 1);
      produce(produced, n, pslot);
      produced += n;
      pslot += n;
      if (pslot >= RR) pslot -= RR;
    }
    // consume: y pass + remap; thread = column cg * 32 + lane, rows U * rg .. + U - 1
    constexpr int kGroups = kElChunk / U;  // row groups per chunk
    for (int task = warp; task < kGroups * (TW / 32); task += kElWarps) {
      const int rg = task % kGroups, cg = task / kGroups;
      const int col = cg * 32 + lane;
      const int r0 = Q + U * rg;  // first output row of this thread
      if (r0 >= yb1) continue;    // (warp-uniform)
      int sbase = (pslot - (produced - (r0 - r))) % RR;  // ring slot of halo row r0 - r
      if (sbase < 0) sbase += RR;
      double dv[2][U];
#pragma unroll
      for (int plane = 0; plane < 2; ++plane) {
        const double* rp = ring + (size_t)plane * RR * RS + col;
        double acc[U], wv[U];
#pragma unroll
        for (int i = 0; i < U; ++i) acc[i] = 0.0;
#pragma unroll
        for (int j = 0; j < U - 1; ++j) wv[j] = wz[j];
        int s_row = sbase;
        for (int mb = 0; mb < M; mb += U) {
#pragma unroll
          for (int s = 0; s < U; ++s) {
            wv[(s + U - 1) % U] = wz[mb + s + U - 1];
            const double v = rp[s_row * RS];
            if (++s_row == RR) s_row = 0;
#pragma unroll
            for (int i = 0; i < U; ++i) acc[i] = __fma_rn(wv[(s + U - 1 - i) % U], v, acc[i]);
          }
        }
#pragma unroll
        for (int i = 0; i < U; ++i) dv[plane][i] = __dmul_rn(a.alpha, acc[i]);
      }
      const int x = x0 + col;
      if (x < W) {
#pragma unroll
        for (int i = 0; i < U; ++i)
          if (r0 + i < yb1) remap(x, r0 + i, dv[0][i], dv[1][i]);
      }
    }
    __syncthreads();  // the next produce overwrites ring rows this chunk read
  }
}

void launch_elastic(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  const size_t smem = elastic_smem(a.g_r);
  if (elastic_strip(a.g_r) == 64) {
    persistent_grid((const void*)k_elastic<8>, kElThreads, smem, a.n_units);  // smem attribute
    k_elastic<8><<<a.n_units, kElThreads, smem, s>>>(a);
  } else {
    persistent_grid((const void*)k_elastic<4>, kElThreads, smem, a.n_units);
    k_elastic<4><<<a.n_units, kElThreads, smem, s>>>(a);
  }
}

}  // namespace alb
