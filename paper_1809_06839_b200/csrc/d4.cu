// d4.cu -- Rot90 / D4 ("a random transformation
// from dihedral group Dih4"): per image the drawn element e (k = e & 3 quarter
// turns, counter-clockwise as displayed, then hflip if e >= 4) composes into
// one signed permutation from output to input coordinates,
//   swap = 0:  x_in = ax x' + bx,  y_in = ay y' + by
//   swap = 1:  x_in = ax y' + bx,  y_in = ay x' + by      (transposing elements)
// Work unit = (image, 64 x 64 output tile).  The tile's source region (also
// 64 x 64, transposed or not) is staged in shared memory with 16-byte aligned
// source runs (pixels as RGBx words, stride 65 = 1 mod 32 so a column walk is
// conflict-free); each output row is then gathered from the stage into a row
// buffer pre-shifted by the destination's 16-byte phase and copied out in
// aligned 16-byte chunks.  Masks (C = 1) take the same path with byte pixels.
#include <type_traits>

#include "stages.cuh"

namespace alb {

constexpr int kD4Threads = 256;
constexpr int kD4TW = 64;           // tile columns
constexpr int kD4TH = 64;           // tile rows
constexpr int kD4Stage = 64 * 65;   // staged pixels (stride 65)

struct SMap {
  int sw, ax, bx, ay, by;
};

// output -> input map of element e on a win x hin input (fired gate), built
// by peeling the ops from the last: hflip in the rotated frame, then the k
// quarter turns (one turn's inverse: x_in = W_in - 1 - y', y_in = x')
__device__ __forceinline__ SMap d4_map(int e, int win, int hin) {
  const int k = e & 3;
  SMap m{0, 1, 0, 1, 0};
  if (e >= 4) {
    const int wk = (k & 1) ? hin : win;
    m.ax = -1;
    m.bx = wk - 1;
  }
  for (int t = k; t >= 1; --t) {
    const int wprev = ((t - 1) & 1) ? hin : win;
    SMap n;
    n.sw = !m.sw;
    n.ax = -m.ay;
    n.bx = wprev - 1 - m.by;
    n.ay = m.ax;
    n.by = m.bx;
    m = n;
  }
  return m;
}

template <int C>
__global__ void __launch_bounds__(kD4Threads) k_d4(StepArgs a) {
  using Px = typename std::conditional<C == 3, uint32_t, uint8_t>::type;
  __shared__ __align__(16) Px stage[kD4Stage + 16];
  __shared__ __align__(16) uint8_t obuf[kD4TH * (kD4TW * C + 16)];
  constexpr int kObp = kD4TW * C + 16;
  const int2 unit = a.units[blockIdx.x];
  const int img = unit.x;
  const alb_image_desc sd = C == 3 ? a.sdesc[img] : a.msdesc[img];
  const alb_image_desc dd = C == 3 ? a.ddesc[img] : a.mddesc[img];
  const uint8_t* simg = (C == 3 ? a.src : a.msrc) + sd.offset;
  uint8_t* dimg = (C == 3 ? a.dst : a.mdst) + dd.offset;
  const int Wo = dd.width, Ho = dd.height, Ws = sd.width, Hs = sd.height;
  const SMap m = fired_of(a.tab, img, a.slot0) ? d4_map((int)prm_of(a.tab, img, a.slot0)[0], Ws, Hs)
                                                : SMap{0, 1, 0, 1, 0};
  const int tx0 = (unit.y & 0xffff) * kD4TW, ty0 = (unit.y >> 16) * kD4TH;
  const int tw = min(kD4TW, Wo - tx0), th = min(kD4TH, Ho - ty0);
  constexpr int S = 65;  // stage stride = 1 mod 32
  // source region of the tile
  const int ua = m.sw ? ty0 : tx0, ub = (m.sw ? ty0 + th : tx0 + tw) - 1;  // feeds x_in
  const int va = m.sw ? tx0 : ty0, vb = (m.sw ? tx0 + tw : ty0 + th) - 1;  // feeds y_in
  const int rx0 = min(m.ax * ua + m.bx, m.ax * ub + m.bx), rw = ub - ua + 1;
  const int ry0 = min(m.ay * va + m.by, m.ay * vb + m.by), rh = vb - va + 1;
  __shared__ int phase[kD4TH];  // destination 16-byte phase of each tile row
  if (threadIdx.x < th)
    phase[threadIdx.x] = (int)((uintptr_t)(dimg + (size_t)(ty0 + threadIdx.x) * dd.pitch + (size_t)tx0 * C) & 15);
  // 1. stage the region: 16-pixel runs whose source bytes are 16-byte aligned
  const int X0 = rx0, X1 = rx0 + rw;
  const int nrun = (rw + 30) >> 4;
  const uint32_t mrh = magic_of((uint32_t)rh);
  for (int it = threadIdx.x; it < rh * nrun; it += kD4Threads) {
    const int k = fdiv(it, mrh), r = it - k * rh;
    const uint8_t* srow = simg + (size_t)(ry0 + r) * sd.pitch;
    const int xa = C == 3 ? (11 * (16 - (int)((uintptr_t)srow & 15))) & 15 : (16 - (int)((uintptr_t)srow & 15)) & 15;
    const int xs = X0 - ((X0 - xa) & 15) + 16 * k;
    if (xs >= X1) continue;
    const uint8_t* p = srow + C * (ptrdiff_t)xs;  // 16-byte aligned
    const uint8_t* lo = srow + C * X0;
    const uint8_t* hi = srow + C * X1;
    uint32_t w[12];
#pragma unroll
    for (int v = 0; v < C; ++v) {
      const uint8_t* q = p + 16 * v;
      uint4 z = make_uint4(0, 0, 0, 0);
      if (q < hi && q + 16 > lo) z = __ldg(reinterpret_cast<const uint4*>(q));
      w[4 * v] = z.x; w[4 * v + 1] = z.y; w[4 * v + 2] = z.z; w[4 * v + 3] = z.w;
    }
    Px* d = stage + r * S + (xs - X0);
    if (xs >= X0 && xs + 16 <= X1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if constexpr (C == 3) d[i] = rgbx_raw(w, i);
        else d[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
      }
    } else {
      const int lo_i = max(X0 - xs, 0), hi_i = min(X1 - xs, 16);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i >= lo_i && i < hi_i) {
          if constexpr (C == 3) d[i] = rgbx_raw(w, i);
          else d[i] = (uint8_t)(w[i >> 2] >> (8 * (i & 3)));
        }
    }
  }
  __syncthreads();
  // 2. gather: output pixel (x', y') of the tile <- stage (x_in - rx0, y_in - ry0);
  // thread = column xl, rows yl0 + 4j: the stage index moves by a constant per row
  {
    const int xl = threadIdx.x & 63, yl0 = threadIdx.x >> 6;
    if (xl < tw) {
      const int xo = tx0 + xl, yo0 = ty0 + yl0;
      int idx, step;
      if (m.sw) {  // x_in from y', y_in from x'
        idx = (m.ay * xo + m.by - ry0) * S + (m.ax * yo0 + m.bx - rx0);
        step = 4 * m.ax;
      } else {
        idx = (m.ay * yo0 + m.by - ry0) * S + (m.ax * xo + m.bx - rx0);
        step = 4 * m.ay * S;
      }
      uint8_t* ob = obuf + yl0 * kObp + C * xl;
      for (int yl = yl0; yl < th; yl += 4, idx += step, ob += 4 * kObp) {
        const Px v = stage[idx];
        uint8_t* o = ob + phase[yl];
        if constexpr (C == 3) {
          o[0] = (uint8_t)v;
          o[1] = (uint8_t)(v >> 8);
          o[2] = (uint8_t)(v >> 16);
        } else {
          o[0] = v;
        }
      }
    }
  }
  __syncthreads();
  // 3. aligned chunk copy-out
  copy_rows_out<C == 3 ? 12 : 4, kD4Threads>(dimg + (size_t)ty0 * dd.pitch + (size_t)tx0 * C, dd.pitch, obuf,
                                             kObp, th, C * tw);
}

void launch_d4(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  if (a.channels == 3) k_d4<3><<<a.n_units, kD4Threads, 0, s>>>(a);
  else k_d4<1><<<a.n_units, kD4Threads, 0, s>>>(a);
}

}  // namespace alb
