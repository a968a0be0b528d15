// affine.cu -- K4 Rotate / ShiftScaleRotate (O7) with fused post
// ops (K10: RandomCrop / Crop / flips on the output coordinates), the
// pointwise stage chain, Normalize output and the nearest-neighbour mask.
//
// Inverse map per warp-output pixel (xw, yw):
//   x_s = cx + (cos*(xw-cx-tx) - sin*(yw-cy-ty)) / s,  likewise y_s,
// written as x_s = A0*xw + A1*yw + A2 with the coefficients formed in fp64.
// Coordinates: an fp64 ANCHOR per 16x16 cell of warp-output coordinates
// (split into integer + fp32 fraction) plus fp32 local offsets (<= 15 px):
// error ~2e-6 px, and a pixel's value depends only on its warp-output
// coordinates, so the fused cfg5 kernel equals the unfused kernel bit for bit.
//
// Work unit = (image, 64x64 output tile); the grid is persistent over
// contiguous unit ranges.  Per tile the source footprint (+ bilinear halo) is
// staged in shared memory as RGBx words with the border resolved per staged
// pixel (reflect-101 or constant fill), so the hot loop has no border logic.
// The staged row stride S is = +-1 (mod 32), picked from the rotation so the
// 32 lanes of a warp (32 consecutive output pixels) hit distinct banks.
// Each lane computes one pixel per row; rows are written with warp-shuffled
// 4-byte stores (warp_store_rgb).  Footprints larger than the staging
// capacity fall back to per-tap global loads.
#include "stages.cuh"

namespace alb {

constexpr int kAfThreads = 256;
constexpr int kTile = 64;
constexpr int kCells = 5;  // 16x16 anchor cells per tile axis (64 px unaligned -> <= 5)

struct AfCoef {
  double A[6];
};

__device__ __forceinline__ AfCoef af_coef(const StepArgs& a, int img) {
  AfCoef c;
  if (!fired_of(a.tab, img, a.slot0)) {  // gate not fired: identity map
    c.A[0] = 1; c.A[1] = 0; c.A[2] = 0; c.A[3] = 0; c.A[4] = 1; c.A[5] = 0;
    return c;
  }
  const alb_op& o = a.ops[a.slot0];
  const double* q = prm_of(a.tab, img, a.slot0);
  double dx = 0.0, dy = 0.0, s = 1.0, th;
  if (o.kind == ALB_SHIFT_SCALE_ROTATE) {
    dx = q[0]; dy = q[1]; s = q[2]; th = q[3];
  } else {
    th = q[0];
  }
  const int W = dim_w(a.tab, img, a.slot0), H = dim_h(a.tab, img, a.slot0);
  const double rad = __ddiv_rn(__dmul_rn(th, 3.141592653589793), 180.0);
  double sn, cs;
  sincos(rad, &sn, &cs);
  const double cx = __ddiv_rn((double)W - 1.0, 2.0), cy = __ddiv_rn((double)H - 1.0, 2.0);
  const double tx = __dmul_rn(dx, (double)W), ty = __dmul_rn(dy, (double)H);
  const double ux = __dadd_rn(cx, tx), uy = __dadd_rn(cy, ty);
  c.A[0] = cs / s;
  c.A[1] = -sn / s;
  c.A[2] = cx - (cs * ux - sn * uy) / s;
  c.A[3] = sn / s;
  c.A[4] = cs / s;
  c.A[5] = cy - (sn * ux + cs * uy) / s;
  return c;
}

__device__ __forceinline__ uint32_t fetch_rgb(const uint8_t* row, int x) {
  const uint8_t* p = row + 3 * x;
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16);
}

struct Anchor {
  int ix, iy;
  float fx, fy;
};

__global__ void __launch_bounds__(kAfThreads) k_affine(StepArgs a) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  StageCtx x;
  init_stages(a, x);
  Anchor* anc = reinterpret_cast<Anchor*>(sm + x.n_lut * kLutWords);
  int* s_geom = reinterpret_cast<int*>(anc + kCells * kCells);  // fx0, fy0, S, fw, fh, staged, cx0, cy0, Sm
  uint32_t* stage = reinterpret_cast<uint32_t*>(s_geom + 16);
  uint8_t* mstage = reinterpret_cast<uint8_t*>(stage + a.unit_size);
  const bool reflect = a.border == ALB_BORDER_REFLECT_101;
  const bool nearest = a.interp == ALB_INTERP_NEAREST;
  const bool has_mask = a.mdst != nullptr;

  int u0, u1;
  unit_range(a.n_units, u0, u1);
  int cur_img = -1;
  AfCoef cf;
  Map1 m;
  int Wo = 0, Ho = 0, tiles_x = 1;
  for (int u = u0; u < u1; ++u) {
    const int2 unit = a.units[u];
    const int img = unit.x;
    __syncthreads();  // previous tile fully consumed
    if (img != cur_img) {
      load_stages(a, img, sm, x, kAfThreads);
      cf = af_coef(a, img);
      Wo = a.normalize ? a.out_w : a.ddesc[img].width;
      Ho = a.normalize ? a.out_h : a.ddesc[img].height;
      m = compose_exact(a.ops, a.tab, img, a.slot0 + 1, a.slot1, Wo, Ho);
      tiles_x = (Wo + kTile - 1) / kTile;
      cur_img = img;
    }
    const alb_image_desc sd = a.sdesc[img];
    const int Ws = sd.width, Hs = sd.height;
    const int tx0 = (unit.y % tiles_x) * kTile, ty0 = (unit.y / tiles_x) * kTile;
    const int tw = min(kTile, Wo - tx0), th = min(kTile, Ho - ty0);
    // warp-output rectangle of the tile
    const int xwa = m.ax * tx0 + m.bx, xwb = m.ax * (tx0 + tw - 1) + m.bx;
    const int ywa = m.ay * ty0 + m.by, ywb = m.ay * (ty0 + th - 1) + m.by;
    const int xw0 = min(xwa, xwb), xw1 = max(xwa, xwb), yw0 = min(ywa, ywb), yw1 = max(ywa, ywb);
    if (threadIdx.x == 0) {
      double lx = 1e300, hx = -1e300, ly = 1e300, hy = -1e300;
      for (int c = 0; c < 4; ++c) {
        const double xw = (c & 1) ? xw1 : xw0, yw = (c & 2) ? yw1 : yw0;
        const double sx = fma(cf.A[0], xw, fma(cf.A[1], yw, cf.A[2]));
        const double sy = fma(cf.A[3], xw, fma(cf.A[4], yw, cf.A[5]));
        lx = fmin(lx, sx); hx = fmax(hx, sx); ly = fmin(ly, sy); hy = fmax(hy, sy);
      }
      const int fx0 = (int)floor(lx) - 1, fx1 = (int)floor(hx) + 2;
      const int fy0 = (int)floor(ly) - 1, fy1 = (int)floor(hy) + 2;
      const int fw = fx1 - fx0 + 1, fh = fy1 - fy0 + 1;
      // bank-friendly stride: lane step is +-(A0 + S*A3) words
      const int want = fabs(cf.A[0] + cf.A[3]) >= fabs(cf.A[0] - cf.A[3]) ? 1 : 31;
      int S = fw + ((want - fw % 32) + 32) % 32;
      const int Sm = (fw + 3) & ~3;
      const bool staged = (long long)S * fh <= a.unit_size && (long long)Sm * fh <= 4LL * a.unit_size / 4;
      s_geom[0] = fx0; s_geom[1] = fy0; s_geom[2] = S; s_geom[3] = fw; s_geom[4] = fh;
      s_geom[5] = staged ? 1 : 0; s_geom[6] = xw0 >> 4; s_geom[7] = yw0 >> 4; s_geom[8] = Sm;
    }
    if (threadIdx.x < kCells * kCells) {
      const int cxa = (xw0 >> 4) + threadIdx.x % kCells, cya = (yw0 >> 4) + threadIdx.x / kCells;
      const double xa = (double)(cxa * 16), ya = (double)(cya * 16);
      const double sx = fma(cf.A[0], xa, fma(cf.A[1], ya, cf.A[2]));
      const double sy = fma(cf.A[3], xa, fma(cf.A[4], ya, cf.A[5]));
      const double fx = floor(sx), fy = floor(sy);
      Anchor an;
      an.ix = (int)fx; an.iy = (int)fy;
      an.fx = (float)(sx - fx); an.fy = (float)(sy - fy);
      anc[threadIdx.x] = an;
    }
    __syncthreads();
    const int fx0 = s_geom[0], fy0 = s_geom[1], S = s_geom[2], fw = s_geom[3], fh = s_geom[4];
    const bool staged = s_geom[5] != 0;
    const int cx0 = s_geom[6], cy0 = s_geom[7], Sm = s_geom[8];
    const uint8_t* simg = a.src + sd.offset;
    const uint8_t* smk = has_mask ? a.msrc + a.msdesc[img].offset : nullptr;
    const int mpitch = has_mask ? a.msdesc[img].pitch : 0;
    if (staged) {
      const int per_row = (fw + 15) / 16;
      for (int it = threadIdx.x; it < fh * per_row; it += kAfThreads) {
        const int r = it / per_row, c16 = (it % per_row) * 16;
        const int sy = fy0 + r;
        int ry = sy;
        bool row_in = sy >= 0 && sy < Hs;
        if (!row_in && reflect) { ry = reflect101(sy, Hs); row_in = true; }
        const int sx0 = fx0 + c16;
        uint32_t* d = stage + r * S + c16;
        const uint8_t* srow = simg + (size_t)ry * sd.pitch;
        if (row_in && sx0 >= 0 && sx0 + 16 <= Ws) {
          uint32_t w[12];
          load_window<12>(srow + (size_t)sx0 * 3, srow, srow + (size_t)Ws * 3, w);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c16 + i < fw) d[i] = rgbx_of(w, i);
        } else {
          for (int i = 0; i < 16 && c16 + i < fw; ++i) {
            const int sx = sx0 + i;
            uint32_t v = a.fill;
            if (row_in) {
              if (sx >= 0 && sx < Ws) v = fetch_rgb(srow, sx);
              else if (reflect) v = fetch_rgb(srow, reflect101(sx, Ws));
            }
            d[i] = v;
          }
        }
        if (has_mask) {
          const uint8_t* mrow = smk + (size_t)ry * mpitch;
          uint8_t* md = mstage + r * Sm + c16;
          for (int i = 0; i < 16 && c16 + i < fw; ++i) {
            const int sx = sx0 + i;
            uint8_t v = (uint8_t)a.mask_fill;
            if (row_in) {
              if (sx >= 0 && sx < Ws) v = mrow[sx];
              else if (reflect) v = mrow[reflect101(sx, Ws)];
            }
            md[i] = v;
          }
        }
      }
      __syncthreads();
    }
    // ---- compute: warp w handles (row, 32-px segment) pairs
    const int nseg = (tw + 31) / 32;
    const float A0f = (float)cf.A[0], A1f = (float)cf.A[1], A3f = (float)cf.A[3], A4f = (float)cf.A[4];
    for (int rs = warp; rs < th * nseg; rs += kAfThreads / 32) {
      const int row = rs / nseg, seg = rs % nseg;
      const int yo = ty0 + row;
      const int xo = tx0 + seg * 32 + lane;
      const int nvalid = min(32, tw - seg * 32);
      const bool act = lane < nvalid;
      const int xw = m.ax * min(xo, Wo - 1) + m.bx, yw = m.ay * yo + m.by;
      const Anchor an = anc[((xw >> 4) - cx0) + kCells * ((yw >> 4) - cy0)];
      const float dxl = (float)(xw & 15), dyl = (float)(yw & 15);
      const float lx = fmaf(A0f, dxl, fmaf(A1f, dyl, an.fx));
      const float ly = fmaf(A3f, dxl, fmaf(A4f, dyl, an.fy));
      uint32_t r, g, b;
      if (nearest) {
        const int tx = an.ix + (int)floorf(lx + 0.5f), ty = an.iy + (int)floorf(ly + 0.5f);
        uint32_t t;
        if (staged) {
          t = stage[(ty - fy0) * S + (tx - fx0)];
        } else if (tx >= 0 && tx < Ws && ty >= 0 && ty < Hs) {
          t = fetch_rgb(simg + (size_t)ty * sd.pitch, tx);
        } else if (reflect) {
          t = fetch_rgb(simg + (size_t)reflect101(ty, Hs) * sd.pitch, reflect101(tx, Ws));
        } else {
          t = a.fill;
        }
        r = t & 0xff; g = (t >> 8) & 0xff; b = (t >> 16) & 0xff;
      } else {
        const float flx = floorf(lx), fly = floorf(ly);
        const float fx = lx - flx, fy = ly - fly;
        const int tx = an.ix + (int)flx, ty = an.iy + (int)fly;
        uint32_t t00, t10, t01, t11;
        if (staged) {
          const uint32_t* p = stage + (ty - fy0) * S + (tx - fx0);
          t00 = p[0]; t10 = p[1]; t01 = p[S]; t11 = p[S + 1];
        } else {
          auto tap = [&](int qx, int qy) -> uint32_t {
            if (qx >= 0 && qx < Ws && qy >= 0 && qy < Hs) return fetch_rgb(simg + (size_t)qy * sd.pitch, qx);
            if (!reflect) return a.fill;
            return fetch_rgb(simg + (size_t)reflect101(qy, Hs) * sd.pitch, reflect101(qx, Ws));
          };
          t00 = tap(tx, ty); t10 = tap(tx + 1, ty); t01 = tap(tx, ty + 1); t11 = tap(tx + 1, ty + 1);
        }
        uint32_t ch[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float p00 = (float)((t00 >> (8 * c)) & 0xff), p10 = (float)((t10 >> (8 * c)) & 0xff);
          const float p01 = (float)((t01 >> (8 * c)) & 0xff), p11 = (float)((t11 >> (8 * c)) & 0xff);
          const float h0 = fmaf(fx, p10 - p00, p00);
          const float h1 = fmaf(fx, p11 - p01, p01);
          const float v = fmaf(fy, h1 - h0, h0);
          ch[c] = (uint32_t)(v + 0.5f);
        }
        r = ch[0]; g = ch[1]; b = ch[2];
      }
      apply_stages(x, sm, lane, r, g, b);
      if (a.normalize) {
        if (act) {
          const size_t plane = (size_t)Ho * Wo;
          float* o = a.nchw + (size_t)img * 3 * plane + (size_t)yo * Wo + xo;
          const float* nl = a.tab.norm_lut;
          o[0] = nl[r]; o[plane] = nl[256 + g]; o[2 * plane] = nl[512 + b];
        }
      } else {
        const alb_image_desc dd = a.ddesc[img];
        uint8_t* drow = a.dst + dd.offset + (size_t)yo * dd.pitch + (size_t)(tx0 + seg * 32) * 3;
        warp_store_rgb(drow, nvalid, r | (g << 8) | (b << 16), lane);
      }
      if (has_mask) {
        const int tx = an.ix + (int)floorf(lx + 0.5f), ty = an.iy + (int)floorf(ly + 0.5f);
        uint8_t v;
        if (staged) {
          v = mstage[(ty - fy0) * Sm + (tx - fx0)];
        } else if (tx >= 0 && tx < Ws && ty >= 0 && ty < Hs) {
          v = smk[(size_t)ty * mpitch + tx];
        } else if (reflect) {
          v = smk[(size_t)reflect101(ty, Hs) * mpitch + reflect101(tx, Ws)];
        } else {
          v = (uint8_t)a.mask_fill;
        }
        if (act) {
          const alb_image_desc mdd = a.mddesc[img];
          a.mdst[mdd.offset + (size_t)yo * mdd.pitch + xo] = v;
        }
      }
    }
  }
}

size_t affine_smem(const StepArgs& a) {
  return (size_t)count_lut_stages(a) * kLutWords * 4 + sizeof(Anchor) * kCells * kCells + 64 +
         (size_t)a.unit_size * 4 + (size_t)a.unit_size;
}

void launch_affine(const StepArgs& a, cudaStream_t s) {
  if (a.n_units <= 0) return;
  const size_t smem = affine_smem(a);
  cudaFuncSetAttribute(k_affine, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1, sms = 148, dev = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_affine, kAfThreads, smem);
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::min(a.n_units, sms * std::max(occ, 1));
  k_affine<<<grid, kAfThreads, smem, s>>>(a);
}

}  // namespace alb
