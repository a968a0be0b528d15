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
// fp32 NCHW run pixel-wise on 48-byte (16-pixel) groups.  Unaligned heads and
// tails, and buffers that are not 16-byte co-aligned, take a per-pixel path.
#include "stages.cuh"

namespace alb {

constexpr int kThreads = 256;
constexpr int kU = 4;  // 16-byte vectors in flight per thread (pure-LUT path)

// kMode: 0 = generic pixel-wise chain, 1 = exactly one LUT stage, 2 = LUT stages only
template <int kMode>
__global__ void __launch_bounds__(kThreads) k_point(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31;
  StageCtx x;
  init_stages(a, x);
  int u0, u1;
  unit_range(a.n_units, u0, u1);
  int cur_img = -1;
  const float* nl = a.tab.norm_lut;
  for (int u = u0; u < u1; ++u) {
    const int2 unit = a.units[u];
    const int img = unit.x;
    if (img != cur_img) {
      __syncthreads();
      load_stages(a, img, sm, x, kThreads);
      __syncthreads();
      cur_img = img;
    }
    const alb_image_desc sd = a.sdesc[img];
    const int W = sd.width, H = sd.height;
    const uint8_t* src;
    uint8_t* dst = nullptr;
    int b0, b1;
    size_t pidx0;  // NCHW plane index of segment byte 0
    if (a.flat) {
      src = a.src + sd.offset;
      if (a.dst) dst = a.dst + a.ddesc[img].offset;
      b0 = unit.y * a.unit_size;
      b1 = min(H * W * 3, b0 + a.unit_size);
      pidx0 = 0;
    } else {
      src = a.src + sd.offset + (size_t)unit.y * sd.pitch;
      if (a.dst) {
        const alb_image_desc dd = a.ddesc[img];
        dst = a.dst + dd.offset + (size_t)unit.y * dd.pitch;
      }
      b0 = 0;
      b1 = W * 3;
      pidx0 = (size_t)unit.y * W;
    }
    const size_t plane = (size_t)H * W;
    float* plane0 = a.normalize ? a.nchw + (size_t)img * 3 * plane : nullptr;

    // aligned body [bA, bE): pixel boundary, 16-byte aligned on both sides
    int bA = b1, bE = b1;
    if (a.vec_ok) {
      int o = b0 + (int)((16 - (((uintptr_t)src + b0) & 15)) & 15);
      while ((o % 3) != 0) o += 16;
      if (o < b1) {
        bA = o;
        bE = bA + ((b1 - bA) / 48) * 48;
      }
    }
    auto scalar_px = [&](int p) {
      uint32_t r = src[3 * p], g = src[3 * p + 1], b = src[3 * p + 2];
      apply_stages(x, sm, lane, r, g, b);
      if (a.normalize) {
        plane0[pidx0 + p] = nl[r];
        plane0[plane + pidx0 + p] = nl[256 + g];
        plane0[2 * plane + pidx0 + p] = nl[512 + b];
      } else {
        dst[3 * p] = (uint8_t)r;
        dst[3 * p + 1] = (uint8_t)g;
        dst[3 * p + 2] = (uint8_t)b;
      }
    };
    for (int p = b0 / 3 + threadIdx.x; p < bA / 3; p += kThreads) scalar_px(p);
    for (int p = bE / 3 + threadIdx.x; p < b1 / 3; p += kThreads) scalar_px(p);
    if (bE <= bA) continue;

    if (kMode != 0) {
      const int nv = (bE - bA) / 16;
      const uint4* s4 = reinterpret_cast<const uint4*>(src + bA);
      uint4* d4 = reinterpret_cast<uint4*>(dst + bA);
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
            const int ph = v % 3;
            const int cb0 = ph * 2048;
            const int cb1 = (ph == 2 ? 0 : ph + 1) * 2048;
            const int cb2 = (ph == 0 ? 2 : ph - 1) * 2048;
            uint32_t w[4] = {in[k].x, in[k].y, in[k].z, in[k].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t o = 0;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int jj = q * 4 + j;
                const int cb = (jj % 3 == 0) ? cb0 : ((jj % 3 == 1) ? cb1 : cb2);
                uint32_t val = (w[q] >> (8 * j)) & 0xffu;
                if (kMode == 1) {
                  val = lut_look(sm, cb, val, lane);
                } else {
                  for (int s = 0; s < x.n_lut; ++s) val = lut_look(sm + s * kLutWords, cb, val, lane);
                }
                o |= val << (8 * j);
              }
              w[q] = o;
            }
            __stcs(d4 + v, make_uint4(w[0], w[1], w[2], w[3]));
          }
        }
      }
    } else {
      const int ng = (bE - bA) / 48;
      for (int gi = threadIdx.x; gi < ng; gi += kThreads) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src + bA + 48 * gi);
        uint32_t w[12];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const uint4 t = __ldcs(s4 + k);
          w[4 * k] = t.x; w[4 * k + 1] = t.y; w[4 * k + 2] = t.z; w[4 * k + 3] = t.w;
        }
        uint32_t o[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) o[k] = 0;
        const int p0 = (bA + 48 * gi) / 3;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          uint32_t r = byte_of(w, 3 * i), g = byte_of(w, 3 * i + 1), b = byte_of(w, 3 * i + 2);
          apply_stages(x, sm, lane, r, g, b);
          if (a.normalize) {
            const size_t pi = pidx0 + p0 + i;
            plane0[pi] = nl[r];
            plane0[plane + pi] = nl[256 + g];
            plane0[2 * plane + pi] = nl[512 + b];
          } else {
            o[(3 * i) >> 2] |= r << (((3 * i) & 3) * 8);
            o[(3 * i + 1) >> 2] |= g << (((3 * i + 1) & 3) * 8);
            o[(3 * i + 2) >> 2] |= b << (((3 * i + 2) & 3) * 8);
          }
        }
        if (!a.normalize) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + bA + 48 * gi);
#pragma unroll
          for (int k = 0; k < 3; ++k)
            __stcs(d4 + k, make_uint4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]));
        }
      }
    }
  }
}

template <int kMode>
static void launch_mode(const StepArgs& a, size_t smem, cudaStream_t s) {
  static int occ_cache[8] = {0};
  const int slot = (int)(smem / (24 * 1024));
  cudaFuncSetAttribute(k_point<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (slot < 8 && occ_cache[slot] == 0) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_point<kMode>, kThreads, smem);
    occ_cache[slot] = occ > 0 ? occ : 1;
  }
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int occ = slot < 8 ? occ_cache[slot] : 1;
  const int grid = std::min(a.n_units, sms * occ);
  k_point<kMode><<<grid, kThreads, smem, s>>>(a);
}

void launch_point(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  const int nl = count_lut_stages(a);
  const bool pure = !a.normalize && nl == a.n_stages && nl > 0;
  const size_t smem = (size_t)nl * kLutWords * 4;
  if (pure && nl == 1) launch_mode<1>(a, smem, s);
  else if (pure) launch_mode<2>(a, smem, s);
  else launch_mode<0>(a, smem, s);
}

}  // namespace alb
