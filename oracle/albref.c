/*
 * albref.c -- CPU ORACLE (test infrastructure only; see albref.h).
 *
 * Plain scalar C in IEEE double, built with -O2 -ffp-contract=off.  Every
 * function follows its definition in the order the definition states it; the
 * citations point at PAPER.md (the method: Table 1 rows at PAPER.md:123-133,
 * the co-transform text at PAPER.md:74-80, the geometry text at PAPER.md:85-87)
 * and at SPEC.md for the formula the paper leaves out, with the DESIGN.md
 * reading (R1..R24, O0..O14) where both are silent.
 *
 * Shares no code with the CUDA path (paper_1809_06839_b200/csrc).
 */
#include "albref.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ O1 RNG */

/* Philox4x32-10: multipliers 0xD2511F53 / 0xCD9E8D57, Weyl bumps
 * 0x9E3779B9 / 0xBB67AE85, ten rounds, key bumped before rounds 2..10.
 * Pinned by the Random123 known-answer vectors (tests/golden/philox_kat.txt). */
void albref_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* u = ((a >> 5) * 2^26 + (b >> 6)) * 2^-53  (O1). */
double albref_u53(uint32_t a, uint32_t b) {
  double hi = (double)(a >> 5);
  double lo = (double)(b >> 6);
  return (hi * 67108864.0 + lo) * (1.0 / 9007199254740992.0);
}

/* draw j of (seed, image, slot): counter (image_lo32, slot, j>>1, TAG_PARAM=0),
 * key (seed_lo32, seed_hi32); words 2(j&1), 2(j&1)+1 (O1). */
double albref_draw(uint64_t seed, uint64_t image_index, int32_t slot, int32_t j) {
  uint32_t ctr[4] = {(uint32_t)image_index, (uint32_t)slot, (uint32_t)(j >> 1), 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t out[4];
  albref_philox4x32_10(ctr, key, out);
  int w = 2 * (j & 1);
  return albref_u53(out[w], out[w + 1]);
}

/* uniform_int(n) = floor(u * n), clamped to n-1. */
static int32_t uniform_int(double u, int32_t n) {
  double f = floor(u * (double)n);
  int32_t k = (int32_t)f;
  if (k > n - 1) k = n - 1;
  return k;
}

/* U(lo, hi) = lo + (hi - lo) * u  (O1). */
static double uniform_range(double lo, double hi, double u) {
  return lo + (hi - lo) * u;
}

/* --------------------------------------------------------- O0 arithmetic */

/* clip_round(v) = min(255, max(0, floor(v + 0.5)))  (R1). */
uint8_t albref_clip_round(double v) {
  double r = floor(v + 0.5);
  if (r < 0.0) return 0;
  if (r > 255.0) return 255;
  return (uint8_t)r;
}

/* reflect-101: -1 -> 1, n -> n-2; periodic with period 2n-2
 * beyond one reflection (reading R7). */
int32_t albref_reflect101(int32_t i, int32_t n) {
  if (n == 1) return 0;
  int64_t period = 2 * (int64_t)n - 2;
  int64_t k = i < 0 ? -(int64_t)i : (int64_t)i;
  k = k % period;
  if (k >= n) k = period - k;
  return (int32_t)k;
}

/* a mod m into [0, m) */
static double fmod_pos(double a, double m) {
  double r = a - m * floor(a / m);
  if (r >= m) r = 0.0;
  if (r < 0.0) r = 0.0;
  return r;
}

/* ---------------------------------------------------------------- O9 HSV */

/* hexcone RGB -> HSV: v = max/255, s = (max-min)/max,
 * h from the dominant-channel sector, ties resolved r > g > b. */
void albref_rgb_to_hsv(double r, double g, double b, double* h, double* s, double* v) {
  double mx = r, mn = r;
  if (g > mx) mx = g;
  if (b > mx) mx = b;
  if (g < mn) mn = g;
  if (b < mn) mn = b;
  double d = mx - mn;
  *v = mx / 255.0;
  *s = mx > 0.0 ? d / mx : 0.0;
  if (d == 0.0) {
    *h = 0.0;
  } else if (mx == r) {
    *h = 60.0 * fmod_pos((g - b) / d, 6.0);
  } else if (mx == g) {
    *h = 60.0 * ((b - r) / d + 2.0);
  } else {
    *h = 60.0 * ((r - g) / d + 4.0);
  }
}

/* hexcone HSV -> RGB (sector decomposition); returns components
 * scaled to [0,255] before rounding. */
void albref_hsv_to_rgb(double h, double s, double v, double* r, double* g, double* b) {
  double C = v * s;
  double hp = h / 60.0;
  double X = C * (1.0 - fabs(fmod_pos(hp, 2.0) - 1.0));
  double m = v - C;
  int sector = (int)floor(hp);
  sector = ((sector % 6) + 6) % 6;
  double r1, g1, b1;
  switch (sector) {
    case 0: r1 = C; g1 = X; b1 = 0.0; break;
    case 1: r1 = X; g1 = C; b1 = 0.0; break;
    case 2: r1 = 0.0; g1 = C; b1 = X; break;
    case 3: r1 = 0.0; g1 = X; b1 = C; break;
    case 4: r1 = X; g1 = 0.0; b1 = C; break;
    default: r1 = C; g1 = 0.0; b1 = X; break;
  }
  *r = 255.0 * (r1 + m);
  *g = 255.0 * (g1 + m);
  *b = 255.0 * (b1 + m);
}

/* ---------------------------------------------------------------- O8 LUT */

static int is_lut_kind(int32_t kind) {
  return kind == ALBREF_BRIGHTNESS || kind == ALBREF_CONTRAST ||
         kind == ALBREF_BRIGHTNESS_CONTRAST || kind == ALBREF_GAMMA ||
         kind == ALBREF_SHIFT_RGB;
}

/* LUT[c][v] of the LUT-type ops (O8):
 *   Brightness  clip_round(v*beta)
 *   Contrast    clip_round(127.5 + (v-127.5)*c)
 *   BC          Contrast_c(Brightness_beta(v))           reading R12
 *   Gamma       clip_round(255*(v/255)^g)
 *   ShiftRGB    clip_round(v + delta_c) */
int albref_build_lut(int32_t kind, const double* prm, uint8_t* lut) {
  if (!is_lut_kind(kind)) return ALBREF_E_UNSUPPORTED;
  for (int c = 0; c < 3; ++c) {
    for (int v = 0; v < 256; ++v) {
      double x = (double)v;
      uint8_t out;
      switch (kind) {
        case ALBREF_BRIGHTNESS: out = albref_clip_round(x * prm[0]); break;
        case ALBREF_CONTRAST: out = albref_clip_round(127.5 + (x - 127.5) * prm[0]); break;
        case ALBREF_BRIGHTNESS_CONTRAST: {
          double t = (double)albref_clip_round(x * prm[0]);
          out = albref_clip_round(127.5 + (t - 127.5) * prm[1]);
          break;
        }
        case ALBREF_GAMMA: out = albref_clip_round(255.0 * pow(x / 255.0, prm[0])); break;
        default: out = albref_clip_round(x + prm[c]); break; /* SHIFT_RGB */
      }
      lut[c * 256 + v] = out;
    }
  }
  return ALBREF_OK;
}

/* Equalize LUT (reading R15): cdf[v] = sum_{u<=v} hist[u]; c_min = hist of the
 * first non-empty bin; D = N - c_min; identity when D == 0; otherwise
 * LUT[v] = floor((2*255*max(cdf[v]-c_min, 0) + D) / (2*D)), i.e. round-half-up
 * of 255*(cdf[v]-c_min)/D in exact integers. */
int albref_equalize_lut(const int64_t* hist, uint8_t* lut) {
  int64_t N = 0;
  for (int v = 0; v < 256; ++v) N += hist[v];
  int64_t c_min = 0;
  for (int v = 0; v < 256; ++v) {
    if (hist[v] > 0) { c_min = hist[v]; break; }
  }
  int64_t D = N - c_min;
  if (D == 0) {
    for (int v = 0; v < 256; ++v) lut[v] = (uint8_t)v;
    return ALBREF_OK;
  }
  int64_t cdf = 0;
  for (int v = 0; v < 256; ++v) {
    cdf += hist[v];
    int64_t num = cdf - c_min;
    if (num < 0) num = 0;
    int64_t q = (2 * 255 * num + D) / (2 * D);
    lut[v] = (uint8_t)q;
  }
  return ALBREF_OK;
}

/* ------------------------------------------------------- validation / shape */

static int is_shape_kind(int32_t k) {
  return k == ALBREF_RANDOM_CROP || k == ALBREF_PAD_TO_SIZE || k == ALBREF_RESIZE ||
         k == ALBREF_RANDOM_SIZED_CROP || k == ALBREF_CROP;
}

static int validate_ops(const albref_op* ops, int32_t n_ops) {
  if (n_ops < 0 || (n_ops > 0 && !ops)) return ALBREF_E_INVALID_ARG;
  for (int32_t k = 0; k < n_ops; ++k) {
    const albref_op* o = &ops[k];
    if (o->kind < 0 || o->kind >= ALBREF_NUM_KINDS) return ALBREF_E_UNKNOWN_OP;
    if (!(o->p >= 0.0 && o->p <= 1.0)) return ALBREF_E_RANGE;
    for (int j = 0; j < 4; ++j)
      if (!(o->lo[j] <= o->hi[j])) return ALBREF_E_RANGE;
    if (is_shape_kind(o->kind) && o->p != 1.0) return ALBREF_E_RANGE; /* R17 */
    if (o->interp != ALBREF_INTERP_NEAREST && o->interp != ALBREF_INTERP_BILINEAR)
      return ALBREF_E_RANGE;
    if (o->border != ALBREF_BORDER_CONSTANT && o->border != ALBREF_BORDER_REFLECT_101)
      return ALBREF_E_RANGE;
    switch (o->kind) {
      case ALBREF_SHIFT_SCALE_ROTATE: if (!(o->lo[2] > 0.0)) return ALBREF_E_RANGE; break;
      case ALBREF_BRIGHTNESS: if (!(o->lo[0] >= 0.0)) return ALBREF_E_RANGE; break;
      case ALBREF_CONTRAST: if (!(o->lo[0] >= 0.0)) return ALBREF_E_RANGE; break;
      case ALBREF_BRIGHTNESS_CONTRAST:
        if (!(o->lo[0] >= 0.0) || !(o->lo[1] >= 0.0)) return ALBREF_E_RANGE;
        break;
      case ALBREF_GAMMA: if (!(o->lo[0] > 0.0)) return ALBREF_E_RANGE; break;
      case ALBREF_RANDOM_CROP: case ALBREF_CROP: case ALBREF_PAD_TO_SIZE: case ALBREF_RESIZE:
        if (o->out_w < 1 || o->out_h < 1) return ALBREF_E_RANGE;
        break;
      case ALBREF_RANDOM_SIZED_CROP:
        if (o->out_w < 1 || o->out_h < 1 || o->min_side < 1 || o->max_side < o->min_side)
          return ALBREF_E_RANGE;
        break;
      case ALBREF_ROT90:
      case ALBREF_D4: { /* integer element range inside the group */
        const double top = o->kind == ALBREF_ROT90 ? 3.0 : 7.0;
        if (!(o->lo[0] >= 0.0 && o->hi[0] <= top) || floor(o->lo[0]) != o->lo[0] ||
            floor(o->hi[0]) != o->hi[0])
          return ALBREF_E_RANGE;
        break;
      }
      case ALBREF_GRID_DISTORTION: /* step factors 1 + U(lo, hi) must stay > 0 */
        if (o->num_steps < 1 || o->num_steps > ALBREF_GRID_MAX_STEPS) return ALBREF_E_RANGE;
        if (!(o->lo[0] > -1.0 && o->hi[0] < 1.0)) return ALBREF_E_RANGE;
        break;
      case ALBREF_ELASTIC: /* fixed alpha >= 0, sigma in (0, 16] (R32) */
        if (o->lo[0] != o->hi[0] || o->lo[1] != o->hi[1]) return ALBREF_E_RANGE;
        if (!(o->lo[0] >= 0.0) || !(o->lo[1] > 0.0 && o->lo[1] <= ALBREF_ELASTIC_MAX_SIGMA))
          return ALBREF_E_RANGE;
        break;
      case ALBREF_NORMALIZE:
        if (k != n_ops - 1 || o->p != 1.0) return ALBREF_E_RANGE;
        for (int c = 0; c < 3; ++c)
          if (!(o->std[c] != 0.0)) return ALBREF_E_RANGE;
        break;
      default: break;
    }
  }
  return ALBREF_OK;
}

static int step_shape(const albref_op* o, int32_t h, int32_t w, int32_t* oh, int32_t* ow) {
  switch (o->kind) {
    case ALBREF_RANDOM_CROP:
      if (o->out_w > w || o->out_h > h) return ALBREF_E_INVALID_ARG;
      *oh = o->out_h; *ow = o->out_w; return ALBREF_OK;
    case ALBREF_CROP:
      if (o->crop_x < 0 || o->crop_y < 0 || o->crop_x + o->out_w > w || o->crop_y + o->out_h > h)
        return ALBREF_E_INVALID_ARG;
      *oh = o->out_h; *ow = o->out_w; return ALBREF_OK;
    case ALBREF_PAD_TO_SIZE:
      if (w > o->out_w || h > o->out_h) return ALBREF_E_INVALID_ARG;
      *oh = o->out_h; *ow = o->out_w; return ALBREF_OK;
    case ALBREF_RESIZE:
      *oh = o->out_h; *ow = o->out_w; return ALBREF_OK;
    case ALBREF_RANDOM_SIZED_CROP: {
      int32_t mside = h < w ? h : w;
      if (o->min_side > mside) return ALBREF_E_INVALID_ARG;
      *oh = o->out_h; *ow = o->out_w; return ALBREF_OK;
    }
    case ALBREF_ROT90:
    case ALBREF_D4: {
      /* an odd number of quarter turns transposes the shape: the output shape
       * must not depend on the draw, so a non-square image needs every
       * outcome (including "gate not fired") to have the same parity */
      int can_odd = 0, can_even = o->p < 1.0;
      for (int32_t e = (int32_t)o->lo[0]; e <= (int32_t)o->hi[0]; ++e) {
        if ((e & 1) != 0) can_odd = 1; else can_even = 1;
      }
      if (can_odd && can_even && h != w) return ALBREF_E_UNSUPPORTED;
      if (can_odd) { *oh = w; *ow = h; } else { *oh = h; *ow = w; }
      return ALBREF_OK;
    }
    default:
      *oh = h; *ow = w; return ALBREF_OK;
  }
}

int albref_output_shape(const albref_op* ops, int32_t n_ops, int32_t in_h, int32_t in_w,
                        int32_t* out_h, int32_t* out_w) {
  int rc = validate_ops(ops, n_ops);
  if (rc) return rc;
  if (in_h < 1 || in_w < 1) return ALBREF_E_SHAPE;
  int32_t h = in_h, w = in_w;
  for (int32_t k = 0; k < n_ops; ++k) {
    rc = step_shape(&ops[k], h, w, &h, &w);
    if (rc) return rc;
  }
  *out_h = h; *out_w = w;
  return ALBREF_OK;
}

/* ---------------------------------------------------------- O1 parameters */

/* Param draws j = 1, 2, ... after the gate (draw 0), in the DESIGN.md O1 table
 * order; h, w are the dims the slot sees. */
static void draw_params(const albref_op* o, uint64_t seed, uint64_t idx, int32_t slot,
                        int32_t h, int32_t w, double* prm) {
  for (int j = 0; j < ALBREF_MAX_PARAMS; ++j) prm[j] = 0.0;
  switch (o->kind) {
    case ALBREF_ROTATE:
    case ALBREF_BRIGHTNESS:
    case ALBREF_CONTRAST:
    case ALBREF_GAMMA:
      prm[0] = uniform_range(o->lo[0], o->hi[0], albref_draw(seed, idx, slot, 1));
      break;
    case ALBREF_BRIGHTNESS_CONTRAST:
      for (int j = 0; j < 2; ++j)
        prm[j] = uniform_range(o->lo[j], o->hi[j], albref_draw(seed, idx, slot, 1 + j));
      break;
    case ALBREF_SHIFT_RGB:
    case ALBREF_SHIFT_HSV:
      for (int j = 0; j < 3; ++j)
        prm[j] = uniform_range(o->lo[j], o->hi[j], albref_draw(seed, idx, slot, 1 + j));
      break;
    case ALBREF_SHIFT_SCALE_ROTATE: /* dx, dy, scale, theta */
      for (int j = 0; j < 4; ++j)
        prm[j] = uniform_range(o->lo[j], o->hi[j], albref_draw(seed, idx, slot, 1 + j));
      break;
    case ALBREF_RANDOM_CROP: /* x0 then y0 */
      prm[0] = (double)uniform_int(albref_draw(seed, idx, slot, 1), w - o->out_w + 1);
      prm[1] = (double)uniform_int(albref_draw(seed, idx, slot, 2), h - o->out_h + 1);
      break;
    case ALBREF_CROP:
      prm[0] = (double)o->crop_x;
      prm[1] = (double)o->crop_y;
      break;
    case ALBREF_ROT90: /* quarter turns, uniform over the integer range */
    case ALBREF_D4:    /* group element, uniform over the integer range */
      prm[0] = o->lo[0] + (double)uniform_int(albref_draw(seed, idx, slot, 1),
                                              (int32_t)(o->hi[0] - o->lo[0]) + 1);
      break;
    case ALBREF_RANDOM_SIZED_CROP: { /* side, x0, y0 (R6) */
      int32_t mside = h < w ? h : w;
      int32_t hi = o->max_side < mside ? o->max_side : mside;
      int32_t side = o->min_side + uniform_int(albref_draw(seed, idx, slot, 1), hi - o->min_side + 1);
      prm[0] = (double)side;
      prm[1] = (double)uniform_int(albref_draw(seed, idx, slot, 2), w - side + 1);
      prm[2] = (double)uniform_int(albref_draw(seed, idx, slot, 3), h - side + 1);
      break;
    }
    default:
      break;
  }
}

int albref_sample_params(const albref_op* ops, int32_t n_ops, uint64_t seed,
                         uint64_t image_index, int32_t in_h, int32_t in_w,
                         double* params, uint8_t* fired) {
  int rc = validate_ops(ops, n_ops);
  if (rc) return rc;
  if (in_h < 1 || in_w < 1) return ALBREF_E_SHAPE;
  int32_t h = in_h, w = in_w;
  for (int32_t k = 0; k < n_ops; ++k) {
    double gate = albref_draw(seed, image_index, k, 0); /* always drawn */
    fired[k] = gate < ops[k].p ? 1 : 0;
    int32_t nh, nw;
    rc = step_shape(&ops[k], h, w, &nh, &nw);
    if (rc) return rc;
    draw_params(&ops[k], seed, image_index, k, h, w, &params[k * ALBREF_MAX_PARAMS]);
    if (ops[k].kind == ALBREF_ROT90 || ops[k].kind == ALBREF_D4) {
      /* the shape follows the drawn element (only square images may differ) */
      nh = h; nw = w;
      if (fired[k] && ((int32_t)params[k * ALBREF_MAX_PARAMS] & 1)) { nh = w; nw = h; }
    }
    if (fired[k]) { h = nh; w = nw; }
  }
  return ALBREF_OK;
}

/* ----------------------------------------------------------- image state */

typedef struct {
  uint8_t* px;      /* [h][w][c] */
  uint8_t* mask;    /* [h][w] or NULL */
  int32_t h, w, c;
  double* box;      /* [n][4] pixel-edge coordinates, unclipped (R18/R19) */
  int32_t* label;
  int32_t nbox;
  /* Nearest-tie candidate sets (tolerance table "Mask nearest", R20), kept
   * only when the caller asks for them (albref_apply_cand): per pixel up to
   * ALBREF_MAX_CAND values that a correct implementation may produce.  They
   * never feed back into px / mask: the oracle's own result is unchanged. */
  int track;
  uint8_t *cpx, *cnpx;   /* [h][w][K][c], [h][w] (0 = any value) */
  uint8_t *cmk, *cnmk;   /* [h][w][K],    [h][w] */
} state_t;

static uint8_t* xalloc(size_t n) {
  return (uint8_t*)malloc(n ? n : 1);
}

/* tap with border policy: reflect-101 remaps, constant substitutes fill
 * (per tap, reading R7).  Returns 1 and sets *xi,*yi when in range. */
static int border_index(int32_t border, int32_t x, int32_t y, int32_t w, int32_t h,
                        int32_t* xi, int32_t* yi) {
  if (x >= 0 && x < w && y >= 0 && y < h) { *xi = x; *yi = y; return 1; }
  if (border == ALBREF_BORDER_REFLECT_101) {
    *xi = albref_reflect101(x, w);
    *yi = albref_reflect101(y, h);
    return 1;
  }
  return 0;
}

/* bilinear weights as O5/O7: v = (1-fy)((1-fx)p00 + fx p10) + fy((1-fx)p01 + fx p11) */
static double bilerp(double p00, double p10, double p01, double p11, double fx, double fy) {
  return (1.0 - fy) * ((1.0 - fx) * p00 + fx * p10) + fy * ((1.0 - fx) * p01 + fx * p11);
}

/* Sample image channel values at real source coordinate (xs, ys) with the
 * affine-op convention (pixel (x,y) at real (x,y)). */
static void sample_affine(const state_t* s, double xs, double ys, int32_t interp,
                          int32_t border, const uint8_t* fill, uint8_t* out) {
  if (interp == ALBREF_INTERP_NEAREST) {
    int32_t xn = (int32_t)floor(xs + 0.5), yn = (int32_t)floor(ys + 0.5);
    int32_t xi, yi;
    for (int c = 0; c < s->c; ++c)
      out[c] = border_index(border, xn, yn, s->w, s->h, &xi, &yi)
                   ? s->px[((size_t)yi * s->w + xi) * s->c + c]
                   : fill[c];
    return;
  }
  double fx0 = floor(xs), fy0 = floor(ys);
  int32_t x0 = (int32_t)fx0, y0 = (int32_t)fy0;
  double fx = xs - fx0, fy = ys - fy0;
  for (int c = 0; c < s->c; ++c) {
    double p[4];
    for (int t = 0; t < 4; ++t) {
      int32_t xi, yi;
      int32_t tx = x0 + (t & 1), ty = y0 + (t >> 1);
      p[t] = border_index(border, tx, ty, s->w, s->h, &xi, &yi)
                 ? (double)s->px[((size_t)yi * s->w + xi) * s->c + c]
                 : (double)fill[c];
    }
    out[c] = albref_clip_round(bilerp(p[0], p[1], p[2], p[3], fx, fy));
  }
}

static uint8_t sample_mask_nearest(const state_t* s, double xs, double ys, int32_t border,
                                   uint8_t mask_fill) {
  int32_t xn = (int32_t)floor(xs + 0.5), yn = (int32_t)floor(ys + 0.5);
  int32_t xi, yi;
  return border_index(border, xn, yn, s->w, s->h, &xi, &yi) ? s->mask[(size_t)yi * s->w + xi]
                                                            : mask_fill;
}

static void replace_px(state_t* s, uint8_t* px, uint8_t* mask, int32_t h, int32_t w) {
  free(s->px);
  s->px = px;
  if (s->mask) { free(s->mask); s->mask = mask; }
  s->h = h; s->w = w;
}

/* ----------------------------------------- nearest-tie candidate sets (R20)
 *
 * SURVEY.md §8(c) tolerance table, "Mask nearest": a nearest sample whose
 * source coordinate lies within ALBREF_TIE_BAND px of a .5 rounding tie may
 * legitimately take either neighbour (fp32 vs fp64 coordinates).  Each pixel
 * of the image and of the mask carries the set of values reachable that way;
 * exact geometric ops move the sets with the pixels, pointwise ops map every
 * member, a bilinear sample resets the set to its own result. */

typedef struct {
  uint8_t *v, *n;  /* [npix][K][c], [npix] */
  int32_t c;
} cset_t;

static cset_t cset_new(size_t npix, int32_t c) {
  cset_t t;
  t.v = xalloc(npix * ALBREF_MAX_CAND * (size_t)c);
  t.n = xalloc(npix);
  t.c = c;
  return t;
}

static void cset_one(cset_t t, size_t i, const uint8_t* val) {
  t.n[i] = 1;
  memcpy(&t.v[i * ALBREF_MAX_CAND * t.c], val, (size_t)t.c);
}

/* union of the source set (sv, sn) into element i (sn == 0: any value) */
static void cset_add(cset_t t, size_t i, const uint8_t* sv, uint8_t sn) {
  if (t.n[i] == 0) return;
  if (sn == 0) { t.n[i] = 0; return; }
  for (int32_t a = 0; a < sn; ++a) {
    const uint8_t* v = &sv[(size_t)a * t.c];
    int32_t have = 0;
    for (int32_t b = 0; b < t.n[i] && !have; ++b)
      have = memcmp(&t.v[(i * ALBREF_MAX_CAND + b) * t.c], v, (size_t)t.c) == 0;
    if (have) continue;
    if (t.n[i] == ALBREF_MAX_CAND) { t.n[i] = 0; return; }
    memcpy(&t.v[(i * ALBREF_MAX_CAND + t.n[i]) * t.c], v, (size_t)t.c);
    t.n[i]++;
  }
}

static void cset_copy(cset_t t, size_t i, const uint8_t* cv, const uint8_t* cn, size_t j) {
  t.n[i] = 1;  /* seed with the first member, then union the rest */
  if (cn[j] == 0) { t.n[i] = 0; return; }
  memcpy(&t.v[i * ALBREF_MAX_CAND * t.c], &cv[j * ALBREF_MAX_CAND * t.c], (size_t)t.c);
  cset_add(t, i, &cv[j * ALBREF_MAX_CAND * t.c], cn[j]);
}

static void cand_init(state_t* s) {
  const size_t n = (size_t)s->h * s->w;
  cset_t a = cset_new(n, s->c);
  for (size_t i = 0; i < n; ++i) cset_one(a, i, &s->px[i * s->c]);
  s->cpx = a.v; s->cnpx = a.n;
  s->cmk = s->cnmk = NULL;
  if (s->mask) {
    cset_t m = cset_new(n, 1);
    for (size_t i = 0; i < n; ++i) cset_one(m, i, &s->mask[i]);
    s->cmk = m.v; s->cnmk = m.n;
  }
}

static void cand_replace(state_t* s, cset_t a, cset_t m) {
  free(s->cpx); free(s->cnpx);
  s->cpx = a.v; s->cnpx = a.n;
  if (s->cmk) { free(s->cmk); free(s->cnmk); s->cmk = m.v; s->cnmk = m.n; }
  else { free(m.v); free(m.n); }
}

/* Exact geometric op: output pixel i takes the sets of input pixel map[i], or
 * the constant fill (map[i] < 0).  Called before replace_px (s = input). */
static void cand_gather(state_t* s, size_t nout, const int64_t* map, const uint8_t* fill,
                        uint8_t mask_fill) {
  cset_t a = cset_new(nout, s->c), m = cset_new(s->cmk ? nout : 1, 1);
  for (size_t i = 0; i < nout; ++i) {
    if (map[i] >= 0) {
      cset_copy(a, i, s->cpx, s->cnpx, (size_t)map[i]);
      if (s->cmk) cset_copy(m, i, s->cmk, s->cnmk, (size_t)map[i]);
    } else {
      cset_one(a, i, fill);
      if (s->cmk) cset_one(m, i, &mask_fill);
    }
  }
  cand_replace(s, a, m);
}

/* The integer taps a nearest sample at coordinate v may take: round_half_up(v),
 * plus the other neighbour when v is within ALBREF_TIE_BAND of k + 0.5. */
static int32_t tie_taps(double v, int32_t* t) {
  const double f = floor(v);
  if (fabs(v - f - 0.5) < ALBREF_TIE_BAND) { t[0] = (int32_t)f; t[1] = (int32_t)f + 1; return 2; }
  t[0] = (int32_t)floor(v + 0.5);
  return 1;
}

/* Candidate sets of a nearest sample at (xs, ys) into output pixel i.
 * clamp_w > 0: taps clamp to the window [0, clamp_w) x [0, clamp_h) offset by
 * (wx0, wy0) (resize, grid); otherwise the border rule applies per tap
 * (affine, elastic) with fill / mask_fill for constant borders. */
static void cand_nearest(const state_t* s, cset_t* a, cset_t* m, size_t i, double xs, double ys,
                         int32_t clamp_w, int32_t clamp_h, int32_t wx0, int32_t wy0,
                         int32_t border, const uint8_t* fill, uint8_t mask_fill) {
  int32_t tx[2], ty[2];
  const int32_t nx = tie_taps(xs, tx), ny = tie_taps(ys, ty);
  if (a) a->n[i] = 1;
  if (m) m->n[i] = 1;
  int first = 1;
  for (int32_t u = 0; u < ny; ++u)
    for (int32_t q = 0; q < nx; ++q) {
      int32_t xi = 0, yi = 0, in;
      if (clamp_w > 0) {
        xi = tx[q] < 0 ? 0 : tx[q] > clamp_w - 1 ? clamp_w - 1 : tx[q];
        yi = ty[u] < 0 ? 0 : ty[u] > clamp_h - 1 ? clamp_h - 1 : ty[u];
        xi += wx0; yi += wy0; in = 1;
      } else {
        in = border_index(border, tx[q], ty[u], s->w, s->h, &xi, &yi);
      }
      const size_t j = (size_t)yi * s->w + xi;
      if (a) {
        const uint8_t* sv = in ? &s->cpx[j * ALBREF_MAX_CAND * s->c] : fill;
        const uint8_t sn = in ? s->cnpx[j] : 1;
        if (first) { if (sn == 0) a->n[i] = 0; else memcpy(&a->v[i * ALBREF_MAX_CAND * s->c], sv, (size_t)s->c); }
        cset_add(*a, i, sv, sn);
      }
      if (m) {
        const uint8_t* sv = in ? &s->cmk[j * ALBREF_MAX_CAND] : &mask_fill;
        const uint8_t sn = in ? s->cnmk[j] : 1;
        if (first) { if (sn == 0) m->n[i] = 0; else m->v[i * ALBREF_MAX_CAND] = *sv; }
        cset_add(*m, i, sv, sn);
      }
      first = 0;
    }
}

/* Candidate sets of an affine-convention sample (affine ops, elastic): the
 * image takes the nearest-tie sets when interpolating nearest, else its own
 * bilinear result; the mask is always nearest. */
static void cand_sample(const state_t* s, cset_t* ca, cset_t* cm, size_t i, double xs, double ys,
                        const albref_op* o, const uint8_t* out) {
  const int nearest = o->interp == ALBREF_INTERP_NEAREST;
  cand_nearest(s, nearest ? ca : NULL, s->mask ? cm : NULL, i, xs, ys, 0, 0, 0, 0, o->border,
               o->fill, o->mask_fill);
  if (!nearest) cset_one(*ca, i, out);
}

/* ---------------------------------------------------- O2 flips, O3/O4 window */

/* HFlip: out[y][x] = in[y][W-1-x]; boxes x' = W - x */
static void op_hflip(state_t* s) {
  uint8_t* px = xalloc((size_t)s->h * s->w * s->c);
  uint8_t* mk = s->mask ? xalloc((size_t)s->h * s->w) : NULL;
  for (int32_t y = 0; y < s->h; ++y)
    for (int32_t x = 0; x < s->w; ++x) {
      for (int c = 0; c < s->c; ++c)
        px[((size_t)y * s->w + x) * s->c + c] = s->px[((size_t)y * s->w + (s->w - 1 - x)) * s->c + c];
      if (mk) mk[(size_t)y * s->w + x] = s->mask[(size_t)y * s->w + (s->w - 1 - x)];
    }
  for (int32_t b = 0; b < s->nbox; ++b) {
    double x0 = s->box[4 * b + 0], x1 = s->box[4 * b + 2];
    s->box[4 * b + 0] = (double)s->w - x1;
    s->box[4 * b + 2] = (double)s->w - x0;
  }
  if (s->track) {
    int64_t* map = (int64_t*)malloc(sizeof(int64_t) * ((size_t)s->h * s->w + 1));
    for (int32_t y = 0; y < s->h; ++y)
      for (int32_t x = 0; x < s->w; ++x) map[(size_t)y * s->w + x] = (int64_t)y * s->w + (s->w - 1 - x);
    cand_gather(s, (size_t)s->h * s->w, map, NULL, 0);
    free(map);
  }
  replace_px(s, px, mk, s->h, s->w);
}

/* VFlip: out[y] = in[H-1-y]; boxes y' = H - y */
static void op_vflip(state_t* s) {
  uint8_t* px = xalloc((size_t)s->h * s->w * s->c);
  uint8_t* mk = s->mask ? xalloc((size_t)s->h * s->w) : NULL;
  for (int32_t y = 0; y < s->h; ++y)
    for (int32_t x = 0; x < s->w; ++x) {
      for (int c = 0; c < s->c; ++c)
        px[((size_t)y * s->w + x) * s->c + c] = s->px[((size_t)(s->h - 1 - y) * s->w + x) * s->c + c];
      if (mk) mk[(size_t)y * s->w + x] = s->mask[(size_t)(s->h - 1 - y) * s->w + x];
    }
  for (int32_t b = 0; b < s->nbox; ++b) {
    double y0 = s->box[4 * b + 1], y1 = s->box[4 * b + 3];
    s->box[4 * b + 1] = (double)s->h - y1;
    s->box[4 * b + 3] = (double)s->h - y0;
  }
  if (s->track) {
    int64_t* map = (int64_t*)malloc(sizeof(int64_t) * ((size_t)s->h * s->w + 1));
    for (int32_t y = 0; y < s->h; ++y)
      for (int32_t x = 0; x < s->w; ++x) map[(size_t)y * s->w + x] = (int64_t)(s->h - 1 - y) * s->w + x;
    cand_gather(s, (size_t)s->h * s->w, map, NULL, 0);
    free(map);
  }
  replace_px(s, px, mk, s->h, s->w);
}

/* Crop window (x0, y0, cw, ch): out[y][x] = in[y0+y][x0+x]; boxes translate
 * (PAPER.md:123); clipping happens at the end (R19). */
static void op_crop(state_t* s, int32_t x0, int32_t y0, int32_t cw, int32_t ch) {
  uint8_t* px = xalloc((size_t)ch * cw * s->c);
  uint8_t* mk = s->mask ? xalloc((size_t)ch * cw) : NULL;
  for (int32_t y = 0; y < ch; ++y)
    for (int32_t x = 0; x < cw; ++x) {
      for (int c = 0; c < s->c; ++c)
        px[((size_t)y * cw + x) * s->c + c] = s->px[((size_t)(y0 + y) * s->w + (x0 + x)) * s->c + c];
      if (mk) mk[(size_t)y * cw + x] = s->mask[(size_t)(y0 + y) * s->w + (x0 + x)];
    }
  for (int32_t b = 0; b < s->nbox; ++b) {
    s->box[4 * b + 0] -= x0; s->box[4 * b + 2] -= x0;
    s->box[4 * b + 1] -= y0; s->box[4 * b + 3] -= y0;
  }
  if (s->track) {
    int64_t* map = (int64_t*)malloc(sizeof(int64_t) * ((size_t)ch * cw + 1));
    for (int32_t y = 0; y < ch; ++y)
      for (int32_t x = 0; x < cw; ++x) map[(size_t)y * cw + x] = (int64_t)(y0 + y) * s->w + (x0 + x);
    cand_gather(s, (size_t)ch * cw, map, NULL, 0);
    free(map);
  }
  replace_px(s, px, mk, ch, cw);
}

/* PadToSize: centred, left = floor((tw-W)/2), top = floor((th-H)/2), constant
 * fill (R8). */
static void op_pad(state_t* s, const albref_op* o) {
  int32_t tw = o->out_w, th = o->out_h;
  int32_t left = (tw - s->w) / 2, top = (th - s->h) / 2;
  uint8_t* px = xalloc((size_t)th * tw * s->c);
  uint8_t* mk = s->mask ? xalloc((size_t)th * tw) : NULL;
  for (int32_t y = 0; y < th; ++y)
    for (int32_t x = 0; x < tw; ++x) {
      int32_t sx = x - left, sy = y - top;
      int inside = sx >= 0 && sx < s->w && sy >= 0 && sy < s->h;
      for (int c = 0; c < s->c; ++c)
        px[((size_t)y * tw + x) * s->c + c] =
            inside ? s->px[((size_t)sy * s->w + sx) * s->c + c] : o->fill[c];
      if (mk) mk[(size_t)y * tw + x] = inside ? s->mask[(size_t)sy * s->w + sx] : o->mask_fill;
    }
  for (int32_t b = 0; b < s->nbox; ++b) {
    s->box[4 * b + 0] += left; s->box[4 * b + 2] += left;
    s->box[4 * b + 1] += top; s->box[4 * b + 3] += top;
  }
  if (s->track) {
    int64_t* map = (int64_t*)malloc(sizeof(int64_t) * ((size_t)th * tw + 1));
    for (int32_t y = 0; y < th; ++y)
      for (int32_t x = 0; x < tw; ++x) {
        int32_t sx = x - left, sy = y - top;
        map[(size_t)y * tw + x] = (sx >= 0 && sx < s->w && sy >= 0 && sy < s->h)
                                      ? (int64_t)sy * s->w + sx : -1;
      }
    cand_gather(s, (size_t)th * tw, map, o->fill, o->mask_fill);
    free(map);
  }
  replace_px(s, px, mk, th, tw);
}

/* ------------------------------------------------------------- O5 resize */

/* Resize of the window [wx0, wx0+ww) x [wy0, wy0+wh) to nw x nh:
 * x_s = (x_d + 0.5) * W / new_w - 0.5, clamped to the window
 * (replicate border, R9); bilinear as O5, nearest = round_half_up(x_s)
 * (SPEC.md:263).  Masks nearest.  Boxes scale (pixel edges). */
static void op_resize_window(state_t* s, int32_t wx0, int32_t wy0, int32_t ww, int32_t wh,
                             int32_t nw, int32_t nh, int32_t interp) {
  uint8_t* px = xalloc((size_t)nh * nw * s->c);
  uint8_t* mk = s->mask ? xalloc((size_t)nh * nw) : NULL;
  cset_t ca = {0}, cm = {0};
  if (s->track) { ca = cset_new((size_t)nh * nw, s->c); cm = cset_new(s->mask ? (size_t)nh * nw : 1, 1); }
  for (int32_t y = 0; y < nh; ++y) {
    double ys = ((double)y + 0.5) * (double)wh / (double)nh - 0.5;
    if (ys < 0.0) ys = 0.0;
    if (ys > (double)(wh - 1)) ys = (double)(wh - 1);
    for (int32_t x = 0; x < nw; ++x) {
      double xs = ((double)x + 0.5) * (double)ww / (double)nw - 0.5;
      if (xs < 0.0) xs = 0.0;
      if (xs > (double)(ww - 1)) xs = (double)(ww - 1);
      uint8_t* o = &px[((size_t)y * nw + x) * s->c];
      int32_t xn = (int32_t)floor(xs + 0.5), yn = (int32_t)floor(ys + 0.5);
      if (interp == ALBREF_INTERP_NEAREST) {
        for (int c = 0; c < s->c; ++c)
          o[c] = s->px[((size_t)(wy0 + yn) * s->w + (wx0 + xn)) * s->c + c];
      } else {
        double fx0 = floor(xs), fy0 = floor(ys);
        int32_t x0 = (int32_t)fx0, y0 = (int32_t)fy0;
        int32_t x1 = x0 + 1 < ww ? x0 + 1 : ww - 1;
        int32_t y1 = y0 + 1 < wh ? y0 + 1 : wh - 1;
        double fx = xs - fx0, fy = ys - fy0;
        for (int c = 0; c < s->c; ++c) {
          double p00 = s->px[((size_t)(wy0 + y0) * s->w + (wx0 + x0)) * s->c + c];
          double p10 = s->px[((size_t)(wy0 + y0) * s->w + (wx0 + x1)) * s->c + c];
          double p01 = s->px[((size_t)(wy0 + y1) * s->w + (wx0 + x0)) * s->c + c];
          double p11 = s->px[((size_t)(wy0 + y1) * s->w + (wx0 + x1)) * s->c + c];
          o[c] = albref_clip_round(bilerp(p00, p10, p01, p11, fx, fy));
        }
      }
      if (mk) mk[(size_t)y * nw + x] = s->mask[(size_t)(wy0 + yn) * s->w + (wx0 + xn)];
      if (s->track) {
        const size_t i = (size_t)y * nw + x;
        const int nearest = interp == ALBREF_INTERP_NEAREST;
        cand_nearest(s, nearest ? &ca : NULL, s->mask ? &cm : NULL, i, xs, ys, ww, wh, wx0, wy0,
                     0, NULL, 0);
        if (!nearest) cset_one(ca, i, o);
      }
    }
  }
  if (s->track) cand_replace(s, ca, cm);
  for (int32_t b = 0; b < s->nbox; ++b) {
    s->box[4 * b + 0] = (s->box[4 * b + 0] - wx0) * (double)nw / (double)ww;
    s->box[4 * b + 2] = (s->box[4 * b + 2] - wx0) * (double)nw / (double)ww;
    s->box[4 * b + 1] = (s->box[4 * b + 1] - wy0) * (double)nh / (double)wh;
    s->box[4 * b + 3] = (s->box[4 * b + 3] - wy0) * (double)nh / (double)wh;
  }
  replace_px(s, px, mk, nh, nw);
}

/* ------------------------------------------------------- O7 affine warps */

/* Rotate / ShiftScaleRotate:
 * centre c = ((W-1)/2, (H-1)/2), t = (dx*W, dy*H), forward p' = c + s R (p-c) + t
 * with R = [[cos, sin], [-sin, cos]] (CCW as displayed, R2); per output pixel
 *   x_s = cx + (cos*(x_d-cx-tx) - sin*(y_d-cy-ty)) / s
 *   y_s = cy + (sin*(x_d-cx-tx) + cos*(y_d-cy-ty)) / s
 * bilinear/nearest with the op's border, masks nearest.
 * Boxes: 4 corners in pixel-centre frame through the forward map, envelope
 * (R18). */
static void op_affine(state_t* s, const albref_op* o, double dx, double dy, double scale,
                      double theta_deg) {
  double th = theta_deg * 3.141592653589793 / 180.0;
  double cs = cos(th), sn = sin(th);
  double cx = ((double)s->w - 1.0) / 2.0, cy = ((double)s->h - 1.0) / 2.0;
  double tx = dx * (double)s->w, ty = dy * (double)s->h;
  uint8_t* px = xalloc((size_t)s->h * s->w * s->c);
  uint8_t* mk = s->mask ? xalloc((size_t)s->h * s->w) : NULL;
  cset_t ca = {0}, cm = {0};
  if (s->track) { ca = cset_new((size_t)s->h * s->w, s->c); cm = cset_new(s->mask ? (size_t)s->h * s->w : 1, 1); }
  for (int32_t y = 0; y < s->h; ++y)
    for (int32_t x = 0; x < s->w; ++x) {
      double ux = (double)x - cx - tx, uy = (double)y - cy - ty;
      double xs = cx + (cs * ux - sn * uy) / scale;
      double ys = cy + (sn * ux + cs * uy) / scale;
      sample_affine(s, xs, ys, o->interp, o->border, o->fill, &px[((size_t)y * s->w + x) * s->c]);
      if (mk) mk[(size_t)y * s->w + x] = sample_mask_nearest(s, xs, ys, o->border, o->mask_fill);
      if (s->track) cand_sample(s, &ca, &cm, (size_t)y * s->w + x, xs, ys, o, &px[((size_t)y * s->w + x) * s->c]);
    }
  if (s->track) cand_replace(s, ca, cm);
  for (int32_t b = 0; b < s->nbox; ++b) {
    double lo_x = 0, lo_y = 0, hi_x = 0, hi_y = 0;
    for (int k = 0; k < 4; ++k) {
      double X = s->box[4 * b + ((k & 1) ? 2 : 0)];
      double Y = s->box[4 * b + ((k & 2) ? 3 : 1)];
      double xc = X - 0.5, yc = Y - 0.5;
      double xp = cx + scale * (cs * (xc - cx) + sn * (yc - cy)) + tx;
      double yp = cy + scale * (-sn * (xc - cx) + cs * (yc - cy)) + ty;
      double Xp = xp + 0.5, Yp = yp + 0.5;
      if (k == 0 || Xp < lo_x) lo_x = Xp;
      if (k == 0 || Xp > hi_x) hi_x = Xp;
      if (k == 0 || Yp < lo_y) lo_y = Yp;
      if (k == 0 || Yp > hi_y) hi_y = Yp;
    }
    s->box[4 * b + 0] = lo_x; s->box[4 * b + 1] = lo_y;
    s->box[4 * b + 2] = hi_x; s->box[4 * b + 3] = hi_y;
  }
  replace_px(s, px, mk, s->h, s->w);
}

/* ------------------------------------------------------ O8-O12 colour ops */

/* Map every member of every image candidate set through a per-pixel op. */
static void cand_map(state_t* s, void (*f)(uint8_t* px, int32_t c, const void* arg), const void* arg) {
  if (!s->track) return;
  for (size_t i = 0; i < (size_t)s->h * s->w; ++i) {
    uint8_t tmp[ALBREF_MAX_CAND * 3];
    const int32_t n = s->cnpx[i];
    if (n == 0) continue;
    memcpy(tmp, &s->cpx[i * ALBREF_MAX_CAND * s->c], (size_t)n * s->c);
    for (int32_t a = 0; a < n; ++a) f(&tmp[a * s->c], s->c, arg);
    cset_t t = {s->cpx, s->cnpx, s->c};
    cset_one(t, i, tmp);
    cset_add(t, i, tmp, (uint8_t)n);
  }
}

static void lut3_px(uint8_t* p, int32_t nc, const void* lut) {
  for (int c = 0; c < nc; ++c) p[c] = ((const uint8_t*)lut)[c * 256 + p[c]];
}

static void apply_lut3(state_t* s, const uint8_t* lut) {
  for (size_t i = 0; i < (size_t)s->h * s->w; ++i)
    for (int c = 0; c < s->c; ++c) s->px[i * s->c + c] = lut[c * 256 + s->px[i * s->c + c]];
  cand_map(s, lut3_px, lut);
}

/* ShiftHSV per pixel: to HSV, h = (h+dh) mod 360,
 * s, v clamped to [0,1], back to RGB with clip_round. */
static void shift_hsv_px(uint8_t* p, int32_t nc, const void* arg) {
  const double dh = ((const double*)arg)[0], ds = ((const double*)arg)[1], dv = ((const double*)arg)[2];
  (void)nc;
  {
    double h, sat, val, r, g, b;
    albref_rgb_to_hsv((double)p[0], (double)p[1], (double)p[2], &h, &sat, &val);
    h = fmod_pos(h + dh, 360.0);
    sat = sat + ds; if (sat < 0.0) sat = 0.0; if (sat > 1.0) sat = 1.0;
    val = val + dv; if (val < 0.0) val = 0.0; if (val > 1.0) val = 1.0;
    albref_hsv_to_rgb(h, sat, val, &r, &g, &b);
    p[0] = albref_clip_round(r);
    p[1] = albref_clip_round(g);
    p[2] = albref_clip_round(b);
  }
}

static void op_shift_hsv(state_t* s, double dh, double ds, double dv) {
  const double d[3] = {dh, ds, dv};
  for (size_t i = 0; i < (size_t)s->h * s->w; ++i) shift_hsv_px(&s->px[i * 3], 3, d);
  cand_map(s, shift_hsv_px, d);
}

/* Grayscale: y = round_half_up(0.299R + 0.587G + 0.114B) in exact integers,
 * floor((299R + 587G + 114B + 500) / 1000), to all 3 channels (
 * PAPER.md:133; R14). */
static void grayscale_px(uint8_t* p, int32_t nc, const void* arg) {
  (void)nc; (void)arg;
  int32_t y = (299 * (int32_t)p[0] + 587 * (int32_t)p[1] + 114 * (int32_t)p[2] + 500) / 1000;
  p[0] = p[1] = p[2] = (uint8_t)y;
}

static void op_grayscale(state_t* s) {
  for (size_t i = 0; i < (size_t)s->h * s->w; ++i) grayscale_px(&s->px[i * 3], 3, NULL);
  cand_map(s, grayscale_px, NULL);
}

/* Equalize per channel (R15). */
static void op_equalize(state_t* s) {
  uint8_t all[768];
  for (int c = 0; c < s->c; ++c) {
    int64_t hist[256];
    uint8_t* lut = &all[c * 256];
    memset(hist, 0, sizeof(hist));
    for (size_t i = 0; i < (size_t)s->h * s->w; ++i) hist[s->px[i * s->c + c]]++;
    albref_equalize_lut(hist, lut);
    for (size_t i = 0; i < (size_t)s->h * s->w; ++i) s->px[i * s->c + c] = lut[s->px[i * s->c + c]];
  }
  cand_map(s, lut3_px, all);
}

/* Normalize to fp32 NCHW: (float)((v/255 - mean_c)/std_c) (R16). */
static void op_normalize(const state_t* s, const albref_op* o, float* out) {
  for (int c = 0; c < 3; ++c)
    for (int32_t y = 0; y < s->h; ++y)
      for (int32_t x = 0; x < s->w; ++x) {
        double v = (double)s->px[((size_t)y * s->w + x) * 3 + c];
        out[((size_t)c * s->h + y) * s->w + x] = (float)((v / 255.0 - o->mean[c]) / o->std[c]);
      }
}

/* -------------------------------------------------- D4 / rot90 */

/* One counter-clockwise (as displayed) quarter turn:
 * out has height W, width H and out[y][x] = in[x][W-1-y].  Boxes in
 * pixel-edge coordinates: a point (X, Y) goes to (Y, W - X), i.e. the
 * normalized (x, y) -> (y, 1 - x) of SPEC.md:196, then corners re-sorted. */
static void op_rot90_once(state_t* s) {
  const int32_t H = s->h, W = s->w, ho = W, wo = H;
  uint8_t* px = xalloc((size_t)ho * wo * s->c);
  uint8_t* mk = s->mask ? xalloc((size_t)ho * wo) : NULL;
  for (int32_t y = 0; y < ho; ++y)
    for (int32_t x = 0; x < wo; ++x) {
      /* in[x][W-1-y]: row x, column W-1-y */
      for (int c = 0; c < s->c; ++c)
        px[((size_t)y * wo + x) * s->c + c] = s->px[((size_t)x * W + (W - 1 - y)) * s->c + c];
      if (mk) mk[(size_t)y * wo + x] = s->mask[(size_t)x * W + (W - 1 - y)];
    }
  for (int32_t b = 0; b < s->nbox; ++b) {
    const double X0 = s->box[4 * b + 0], Y0 = s->box[4 * b + 1];
    const double X1 = s->box[4 * b + 2], Y1 = s->box[4 * b + 3];
    s->box[4 * b + 0] = Y0;
    s->box[4 * b + 2] = Y1;
    s->box[4 * b + 1] = (double)W - X1;
    s->box[4 * b + 3] = (double)W - X0;
  }
  if (s->track) {
    int64_t* map = (int64_t*)malloc(sizeof(int64_t) * ((size_t)ho * wo + 1));
    for (int32_t y = 0; y < ho; ++y)
      for (int32_t x = 0; x < wo; ++x) map[(size_t)y * wo + x] = (int64_t)x * W + (W - 1 - y);
    cand_gather(s, (size_t)ho * wo, map, NULL, 0);
    free(map);
  }
  replace_px(s, px, mk, ho, wo);
}

/* rot90 by k quarter turns = k single turns */
static void op_rot90(state_t* s, int32_t k) {
  for (int32_t i = 0; i < (k & 3); ++i) op_rot90_once(s);
}

/* D4 element e: e in {r^0..r^3, h o r^0..h o r^3}, r = rot90(1),
 * h = hflip; h o r^k applies r^k first, then h. */
static void op_d4(state_t* s, int32_t e) {
  op_rot90(s, e & 3);
  if (e >= 4) op_hflip(s);
}

/* ------------------------------------------- GridDistortion */

/* Reading R31.  Destination knots d_i = i (L-1)/n, i = 0..n; the
 * cells get lengths proportional to the step factors f_0..f_{n-1} rescaled to
 * the span L-1 ("rescaled to preserve total span"):
 *   c_0 = 0, c_{i+1} = c_i + f_i, S = c_n,  s_i = (L-1) c_i / S.
 * The map is kept as a displacement field ("converts to
 * DisplacementField"): e_i = s_i - d_i at the knots (e_0 = e_n = 0), linear in
 * between, so for destination x with u = x n / (L-1), i = min(floor(u), n-1),
 * t = u - i:
 *   src(x) = x + (e_i + t (e_{i+1} - e_i)),  clamped to [0, L-1].
 * f_n is drawn (SPEC.md:332 draws n+1 factors per axis) but no cell uses it. */
int albref_grid_axis(int32_t L, int32_t n, const double* f, double* src) {
  if (n < 1 || n > ALBREF_GRID_MAX_STEPS || L < 1) return ALBREF_E_RANGE;
  for (int32_t i = 0; i < n; ++i)
    if (!(f[i] > 0.0)) return ALBREF_E_RANGE;
  if (L == 1) { src[0] = 0.0; return ALBREF_OK; }
  double c[ALBREF_GRID_MAX_STEPS + 1], e[ALBREF_GRID_MAX_STEPS + 1];
  c[0] = 0.0;
  for (int32_t i = 0; i < n; ++i) c[i + 1] = c[i] + f[i];
  const double S = c[n], span = (double)(L - 1);
  e[0] = 0.0;
  e[n] = 0.0;
  for (int32_t i = 1; i < n; ++i) e[i] = span * c[i] / S - span * (double)i / (double)n;
  for (int32_t x = 0; x < L; ++x) {
    const double u = (double)x * (double)n / span;
    int32_t i = (int32_t)floor(u);
    if (i > n - 1) i = n - 1;
    const double t = u - (double)i;
    double v = (double)x + (e[i] + t * (e[i + 1] - e[i]));
    if (v < 0.0) v = 0.0;
    if (v > span) v = span;
    src[x] = v;
  }
  return ALBREF_OK;
}

/* Remap with the separable maps (mx, my): bilinear taps (x0, min(x0+1, W-1)),
 * as O5 (the maps stay inside the image, so no border rule is reached);
 * nearest = round_half_up; masks nearest. */
static void op_grid(state_t* s, const albref_op* o, uint64_t seed, uint64_t idx, int32_t slot) {
  const int32_t n = o->num_steps;
  double fx[ALBREF_GRID_MAX_STEPS + 1], fy[ALBREF_GRID_MAX_STEPS + 1];
  for (int32_t i = 0; i <= n; ++i) { /* x factors j = 1..n+1, then y factors */
    fx[i] = 1.0 + uniform_range(o->lo[0], o->hi[0], albref_draw(seed, idx, slot, 1 + i));
    fy[i] = 1.0 + uniform_range(o->lo[0], o->hi[0], albref_draw(seed, idx, slot, n + 2 + i));
  }
  double* mx = (double*)malloc(sizeof(double) * s->w);
  double* my = (double*)malloc(sizeof(double) * s->h);
  albref_grid_axis(s->w, n, fx, mx);
  albref_grid_axis(s->h, n, fy, my);
  uint8_t* px = xalloc((size_t)s->h * s->w * s->c);
  uint8_t* mk = s->mask ? xalloc((size_t)s->h * s->w) : NULL;
  cset_t ca = {0}, cm = {0};
  if (s->track) { ca = cset_new((size_t)s->h * s->w, s->c); cm = cset_new(s->mask ? (size_t)s->h * s->w : 1, 1); }
  for (int32_t y = 0; y < s->h; ++y) {
    const double ys = my[y];
    for (int32_t x = 0; x < s->w; ++x) {
      const double xs = mx[x];
      uint8_t* out = &px[((size_t)y * s->w + x) * s->c];
      const int32_t xn = (int32_t)floor(xs + 0.5), yn = (int32_t)floor(ys + 0.5);
      if (o->interp == ALBREF_INTERP_NEAREST) {
        for (int c = 0; c < s->c; ++c) out[c] = s->px[((size_t)yn * s->w + xn) * s->c + c];
      } else {
        const double fx0 = floor(xs), fy0 = floor(ys);
        const int32_t x0 = (int32_t)fx0, y0 = (int32_t)fy0;
        const int32_t x1 = x0 + 1 < s->w ? x0 + 1 : s->w - 1;
        const int32_t y1 = y0 + 1 < s->h ? y0 + 1 : s->h - 1;
        const double ax = xs - fx0, ay = ys - fy0;
        for (int c = 0; c < s->c; ++c) {
          double p00 = s->px[((size_t)y0 * s->w + x0) * s->c + c];
          double p10 = s->px[((size_t)y0 * s->w + x1) * s->c + c];
          double p01 = s->px[((size_t)y1 * s->w + x0) * s->c + c];
          double p11 = s->px[((size_t)y1 * s->w + x1) * s->c + c];
          out[c] = albref_clip_round(bilerp(p00, p10, p01, p11, ax, ay));
        }
      }
      if (mk) mk[(size_t)y * s->w + x] = s->mask[(size_t)yn * s->w + xn];
      if (s->track) {
        const size_t i = (size_t)y * s->w + x;
        const int nearest = o->interp == ALBREF_INTERP_NEAREST;
        cand_nearest(s, nearest ? &ca : NULL, s->mask ? &cm : NULL, i, xs, ys, s->w, s->h, 0, 0,
                     0, NULL, 0);
        if (!nearest) cset_one(ca, i, out);
      }
    }
  }
  if (s->track) cand_replace(s, ca, cm);
  free(mx);
  free(my);
  replace_px(s, px, mk, s->h, s->w);
}

/* ------------------------------------------ ElasticTransform */

/* Reading R32: g_k = exp(-k^2 / (2 sigma^2)), k = -r..r, r = ceil(3 sigma),
 * divided by their sum (accumulated in ascending k) -- SPEC.md:341. */
int albref_gauss_kernel(double sigma, double* w) {
  if (!(sigma > 0.0 && sigma <= ALBREF_ELASTIC_MAX_SIGMA)) return ALBREF_E_RANGE;
  const int32_t r = (int32_t)ceil(3.0 * sigma);
  double sum = 0.0;
  for (int32_t k = -r; k <= r; ++k) {
    w[k + r] = exp(-(double)(k * k) / (2.0 * sigma * sigma));
    sum += w[k + r];
  }
  for (int32_t k = 0; k <= 2 * r; ++k) w[k] /= sum;
  return r;
}

/* raw planes u, v ~ U(-1, 1) per pixel, row-major, the u plane
 * fully first (draw j = 1 + p for u, 1 + h w + p for v, p = y w + x); each
 * convolved with the kernel along x, then along y (reflect-101 edges),
 * accumulated in ascending k as acc = acc + w * x (IEEE double, no
 * contraction: SURVEY.md §8(c) arithmetic rules); then scaled by alpha. */
int albref_elastic_field(int32_t h, int32_t w, double alpha, double sigma, uint64_t seed,
                         uint64_t image_index, int32_t slot, double* dx, double* dy) {
  double g[2 * 48 + 1];
  const int32_t r = albref_gauss_kernel(sigma, g);
  if (r < 0) return r;
  if (h < 1 || w < 1) return ALBREF_E_SHAPE;
  const size_t n = (size_t)h * w;
  double* raw = (double*)malloc(sizeof(double) * n);
  double* bx = (double*)malloc(sizeof(double) * n);
  for (int plane = 0; plane < 2; ++plane) {
    double* d = plane == 0 ? dx : dy;
    for (size_t p = 0; p < n; ++p)
      raw[p] = uniform_range(-1.0, 1.0,
                             albref_draw(seed, image_index, slot, (int32_t)(1 + plane * n + p)));
    for (int32_t y = 0; y < h; ++y)
      for (int32_t x = 0; x < w; ++x) {
        double acc = 0.0;
        for (int32_t k = -r; k <= r; ++k)
          acc = acc + g[k + r] * raw[(size_t)y * w + albref_reflect101(x + k, w)];
        bx[(size_t)y * w + x] = acc;
      }
    for (int32_t y = 0; y < h; ++y)
      for (int32_t x = 0; x < w; ++x) {
        double acc = 0.0;
        for (int32_t k = -r; k <= r; ++k)
          acc = acc + g[k + r] * bx[(size_t)albref_reflect101(y + k, h) * w + x];
        d[(size_t)y * w + x] = alpha * acc;
      }
  }
  free(raw);
  free(bx);
  return ALBREF_OK;
}

/* Remap at source (x + dx, y + dy) with the op's interpolation
 * and border, exactly as the affine ops sample (O7); masks nearest. */
static void op_elastic(state_t* s, const albref_op* o, uint64_t seed, uint64_t idx, int32_t slot) {
  const size_t n = (size_t)s->h * s->w;
  double* dx = (double*)malloc(sizeof(double) * n);
  double* dy = (double*)malloc(sizeof(double) * n);
  albref_elastic_field(s->h, s->w, o->lo[0], o->lo[1], seed, idx, slot, dx, dy);
  uint8_t* px = xalloc(n * s->c);
  uint8_t* mk = s->mask ? xalloc(n) : NULL;
  cset_t ca = {0}, cm = {0};
  if (s->track) { ca = cset_new(n, s->c); cm = cset_new(s->mask ? n : 1, 1); }
  for (int32_t y = 0; y < s->h; ++y)
    for (int32_t x = 0; x < s->w; ++x) {
      const size_t p = (size_t)y * s->w + x;
      const double xs = (double)x + dx[p], ys = (double)y + dy[p];
      sample_affine(s, xs, ys, o->interp, o->border, o->fill, &px[p * s->c]);
      if (mk) mk[p] = sample_mask_nearest(s, xs, ys, o->border, o->mask_fill);
      if (s->track) cand_sample(s, &ca, &cm, p, xs, ys, o, &px[p * s->c]);
    }
  if (s->track) cand_replace(s, ca, cm);
  free(dx);
  free(dy);
  replace_px(s, px, mk, s->h, s->w);
}

/* ---------------------------------------------------------- O14 apply */

static int apply_impl(const albref_op* ops, int32_t n_ops, uint64_t seed, uint64_t image_index,
                      const uint8_t* img, int32_t h, int32_t w, int32_t channels,
                      const uint8_t* mask,
                      const float* boxes, const int32_t* labels, int32_t n_boxes,
                      float min_visibility,
                      uint8_t* img_out, float* nchw_out, uint8_t* mask_out,
                      float* boxes_out, int32_t* labels_out, int32_t* n_boxes_out,
                      uint8_t* cand_img, uint8_t* cand_img_n, uint8_t* cand_mask,
                      uint8_t* cand_mask_n) {
  int rc = validate_ops(ops, n_ops);
  if (rc) return rc;
  if (h < 1 || w < 1) return ALBREF_E_SHAPE;
  if (channels != 1 && channels != 3) return ALBREF_E_UNSUPPORTED;
  if (!img) return ALBREF_E_INVALID_ARG;
  if (n_boxes < 0 || (n_boxes > 0 && (!boxes || !boxes_out || !n_boxes_out)))
    return ALBREF_E_INVALID_ARG;
  for (int32_t k = 0; k < n_ops; ++k) {
    int32_t kd = ops[k].kind;
    if ((kd == ALBREF_GRID_DISTORTION || kd == ALBREF_ELASTIC) && n_boxes > 0)
      return ALBREF_E_UNSUPPORTED; /* boxes under free-form warps */
    if (channels != 3 && (kd == ALBREF_SHIFT_RGB || kd == ALBREF_SHIFT_HSV ||
                          kd == ALBREF_GRAYSCALE || kd == ALBREF_NORMALIZE))
      return ALBREF_E_UNSUPPORTED;
  }
  int ends_norm = n_ops > 0 && ops[n_ops - 1].kind == ALBREF_NORMALIZE;
  if (ends_norm ? !nchw_out : !img_out) return ALBREF_E_INVALID_ARG;

  /* all params first: validation is atomic */
  double* prm = (double*)malloc(sizeof(double) * ALBREF_MAX_PARAMS * (n_ops ? n_ops : 1));
  uint8_t* fired = xalloc((size_t)n_ops);
  rc = albref_sample_params(ops, n_ops, seed, image_index, h, w, prm, fired);
  if (rc) { free(prm); free(fired); return rc; }

  state_t s;
  s.h = h; s.w = w; s.c = channels;
  s.px = xalloc((size_t)h * w * channels);
  memcpy(s.px, img, (size_t)h * w * channels);
  s.mask = NULL;
  if (mask) { s.mask = xalloc((size_t)h * w); memcpy(s.mask, mask, (size_t)h * w); }
  s.track = cand_img != NULL && cand_img_n != NULL;
  s.cpx = s.cnpx = s.cmk = s.cnmk = NULL;
  if (s.track) cand_init(&s);
  s.nbox = n_boxes;
  s.box = (double*)malloc(sizeof(double) * 4 * (n_boxes ? n_boxes : 1));
  s.label = (int32_t*)malloc(sizeof(int32_t) * (n_boxes ? n_boxes : 1));
  for (int32_t b = 0; b < n_boxes; ++b) {
    s.box[4 * b + 0] = (double)boxes[4 * b + 0] * (double)w;
    s.box[4 * b + 1] = (double)boxes[4 * b + 1] * (double)h;
    s.box[4 * b + 2] = (double)boxes[4 * b + 2] * (double)w;
    s.box[4 * b + 3] = (double)boxes[4 * b + 3] * (double)h;
    s.label[b] = labels ? labels[b] : 0;
  }

  for (int32_t k = 0; k < n_ops; ++k) {
    if (!fired[k]) continue; /* apply iff gate < p */
    const albref_op* o = &ops[k];
    const double* q = &prm[k * ALBREF_MAX_PARAMS];
    uint8_t lut[768];
    switch (o->kind) {
      case ALBREF_HFLIP: op_hflip(&s); break;
      case ALBREF_VFLIP: op_vflip(&s); break;
      case ALBREF_ROTATE: op_affine(&s, o, 0.0, 0.0, 1.0, q[0]); break;
      case ALBREF_SHIFT_SCALE_ROTATE: op_affine(&s, o, q[0], q[1], q[2], q[3]); break;
      case ALBREF_RANDOM_CROP:
      case ALBREF_CROP:
        op_crop(&s, (int32_t)q[0], (int32_t)q[1], o->out_w, o->out_h);
        break;
      case ALBREF_PAD_TO_SIZE: op_pad(&s, o); break;
      case ALBREF_RESIZE: op_resize_window(&s, 0, 0, s.w, s.h, o->out_w, o->out_h, o->interp); break;
      case ALBREF_RANDOM_SIZED_CROP: {
        int32_t side = (int32_t)q[0];
        op_resize_window(&s, (int32_t)q[1], (int32_t)q[2], side, side, o->out_w, o->out_h, o->interp);
        break;
      }
      case ALBREF_BRIGHTNESS: case ALBREF_CONTRAST: case ALBREF_BRIGHTNESS_CONTRAST:
      case ALBREF_GAMMA: case ALBREF_SHIFT_RGB:
        albref_build_lut(o->kind, q, lut);
        apply_lut3(&s, lut);
        break;
      case ALBREF_SHIFT_HSV: op_shift_hsv(&s, q[0], q[1], q[2]); break;
      case ALBREF_GRAYSCALE: op_grayscale(&s); break;
      case ALBREF_EQUALIZE: op_equalize(&s); break;
      case ALBREF_NORMALIZE: op_normalize(&s, o, nchw_out); break;
      case ALBREF_ROT90: op_rot90(&s, (int32_t)q[0]); break;
      case ALBREF_D4: op_d4(&s, (int32_t)q[0]); break;
      case ALBREF_GRID_DISTORTION: op_grid(&s, o, seed, image_index, k); break;
      case ALBREF_ELASTIC: op_elastic(&s, o, seed, image_index, k); break;
      default: break;
    }
  }

  if (!ends_norm) memcpy(img_out, s.px, (size_t)s.h * s.w * s.c);
  if (mask && mask_out) memcpy(mask_out, s.mask, (size_t)s.h * s.w);
  if (s.track) {
    const size_t np = (size_t)s.h * s.w;
    memcpy(cand_img, s.cpx, np * ALBREF_MAX_CAND * s.c);
    memcpy(cand_img_n, s.cnpx, np);
    if (mask && cand_mask && cand_mask_n) {
      memcpy(cand_mask, s.cmk, np * ALBREF_MAX_CAND);
      memcpy(cand_mask_n, s.cnmk, np);
    }
  }

  /* boxes: clip the final unclipped envelope to the image, keep iff non-empty
   * and clipped area >= min_visibility * unclipped area (R19), stable. */
  if (n_boxes_out) {
    int32_t kept = 0;
    for (int32_t b = 0; b < s.nbox; ++b) {
      double X0 = s.box[4 * b + 0], Y0 = s.box[4 * b + 1];
      double X1 = s.box[4 * b + 2], Y1 = s.box[4 * b + 3];
      double area = (X1 - X0) * (Y1 - Y0);
      double cx0 = X0 < 0.0 ? 0.0 : X0, cy0 = Y0 < 0.0 ? 0.0 : Y0;
      double cx1 = X1 > (double)s.w ? (double)s.w : X1;
      double cy1 = Y1 > (double)s.h ? (double)s.h : Y1;
      if (!(cx1 > cx0 && cy1 > cy0)) continue;
      double carea = (cx1 - cx0) * (cy1 - cy0);
      if (!(carea >= (double)min_visibility * area)) continue;
      boxes_out[4 * kept + 0] = (float)(cx0 / (double)s.w);
      boxes_out[4 * kept + 1] = (float)(cy0 / (double)s.h);
      boxes_out[4 * kept + 2] = (float)(cx1 / (double)s.w);
      boxes_out[4 * kept + 3] = (float)(cy1 / (double)s.h);
      if (labels_out) labels_out[kept] = s.label[b];
      kept++;
    }
    *n_boxes_out = kept;
  }

  free(s.px); free(s.mask); free(s.box); free(s.label); free(prm); free(fired);
  free(s.cpx); free(s.cnpx); free(s.cmk); free(s.cnmk);
  return ALBREF_OK;
}

int albref_apply(const albref_op* ops, int32_t n_ops, uint64_t seed, uint64_t image_index,
                 const uint8_t* img, int32_t h, int32_t w, int32_t channels,
                 const uint8_t* mask,
                 const float* boxes, const int32_t* labels, int32_t n_boxes,
                 float min_visibility,
                 uint8_t* img_out, float* nchw_out, uint8_t* mask_out,
                 float* boxes_out, int32_t* labels_out, int32_t* n_boxes_out) {
  return apply_impl(ops, n_ops, seed, image_index, img, h, w, channels, mask, boxes, labels,
                    n_boxes, min_visibility, img_out, nchw_out, mask_out, boxes_out, labels_out,
                    n_boxes_out, NULL, NULL, NULL, NULL);
}

int albref_apply_cand(const albref_op* ops, int32_t n_ops, uint64_t seed, uint64_t image_index,
                      const uint8_t* img, int32_t h, int32_t w, int32_t channels,
                      const uint8_t* mask, uint8_t* img_out, float* nchw_out, uint8_t* mask_out,
                      uint8_t* cand_img, uint8_t* cand_img_n, uint8_t* cand_mask,
                      uint8_t* cand_mask_n) {
  if (!cand_img || !cand_img_n || (mask && (!cand_mask || !cand_mask_n)))
    return ALBREF_E_INVALID_ARG;
  return apply_impl(ops, n_ops, seed, image_index, img, h, w, channels, mask, NULL, NULL, 0, 0.0f,
                    img_out, nchw_out, mask_out, NULL, NULL, NULL, cand_img, cand_img_n,
                    cand_mask, cand_mask_n);
}
