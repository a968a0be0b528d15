/*
 * albref.h -- CPU ORACLE for the augmentation hot path of arXiv 1809.06839
 * ("Albumentations: fast and flexible image augmentations").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1809_06839_b200/, include/alb_b200.h) never links,
 * imports or calls it, and shares no source with it.
 *
 * What it computes: each transform exactly as defined in DESIGN.md "Readings"
 * (the paper names the transforms -- PAPER.md:123-133, Table 1; PAPER.md:64,
 * 76, 85-87 -- but gives no formulas; the formulas follow SPEC.md where it has
 * one and the numbered readings R1..R24 of DESIGN.md otherwise).  Plain scalar
 * C, IEEE double, compiled with -O2 -ffp-contract=off (no FMA contraction), no
 * blocking, fusion or reordering.  One image per call.
 *
 * Layout: images are packed HWC uint8 (pitch = width*channels), RGB order,
 * x = column, y = row, origin top-left.  Masks are packed HxW
 * uint8.  Boxes are normalized xyxy float32 (reading R18).
 *
 * Every function returns 0 on success or a negative ALBREF_E_* code.
 */
#ifndef ALBREF_H
#define ALBREF_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* op kinds (the numbering is part of the written contract in DESIGN.md) */
enum {
  ALBREF_HFLIP = 0, ALBREF_VFLIP = 1, ALBREF_ROTATE = 2, ALBREF_SHIFT_SCALE_ROTATE = 3,
  ALBREF_RANDOM_CROP = 4, ALBREF_PAD_TO_SIZE = 5, ALBREF_RESIZE = 6,
  ALBREF_RANDOM_SIZED_CROP = 7, ALBREF_BRIGHTNESS = 8, ALBREF_CONTRAST = 9,
  ALBREF_BRIGHTNESS_CONTRAST = 10, ALBREF_GAMMA = 11, ALBREF_SHIFT_RGB = 12,
  ALBREF_SHIFT_HSV = 13, ALBREF_GRAYSCALE = 14, ALBREF_EQUALIZE = 15,
  ALBREF_NORMALIZE = 16, ALBREF_CROP = 17,
  ALBREF_ROT90 = 18,  /* SPEC.md:193-201; k quarter turns, k in [lo[0], hi[0]] */
  ALBREF_D4 = 19,     /* SPEC.md:202-210; element e in [lo[0], hi[0]] of 0..7 */
  ALBREF_GRID_DISTORTION = 20, /* SPEC.md:329-337; Fig. 4: factors 1 + U(lo[0], hi[0]) */
  ALBREF_ELASTIC = 21,         /* SPEC.md:338-346; alpha = lo[0], sigma = lo[1] */
  ALBREF_NUM_KINDS = 22
};
enum { ALBREF_INTERP_NEAREST = 0, ALBREF_INTERP_BILINEAR = 1 };
enum { ALBREF_BORDER_CONSTANT = 0, ALBREF_BORDER_REFLECT_101 = 1 };
enum {
  ALBREF_OK = 0, ALBREF_E_INVALID_ARG = -1, ALBREF_E_UNKNOWN_OP = -2, ALBREF_E_RANGE = -3,
  ALBREF_E_SHAPE = -4, ALBREF_E_UNSUPPORTED = -5
};

/* One transform of a pipeline (SPEC.md:470-474 TransformSpec).  Continuous
 * parameter j is drawn as lo[j] + (hi[j]-lo[j])*u (O1). */
typedef struct {
  int32_t kind;
  double p;                 /* application probability, [0,1]              */
  double lo[4], hi[4];      /* per-parameter uniform ranges                 */
  int32_t out_w, out_h;     /* RandomCrop/Crop/PadToSize/Resize/RSC size    */
  int32_t min_side, max_side; /* RandomSizedCrop side range (pixels, R6)    */
  int32_t crop_x, crop_y;   /* Crop window origin                           */
  int32_t interp, border;   /* ALBREF_INTERP_*, ALBREF_BORDER_*             */
  uint8_t fill[3], mask_fill;
  double mean[3], std[3];   /* Normalize                                    */
  int32_t num_steps;        /* GridDistortion cells per axis, [1, 32]       */
  int32_t reserved;
} albref_op;

#define ALBREF_GRID_MAX_STEPS 32
#define ALBREF_ELASTIC_MAX_SIGMA 16.0 /* radius ceil(3 sigma) <= 48 (reading R32) */

#define ALBREF_MAX_PARAMS 8

/* Philox4x32-10 (Salmon et al., SC'11; O1). */
void albref_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* u = ((a>>5)*2^26 + (b>>6)) * 2^-53, exact double in [0,1). */
double albref_u53(uint32_t a, uint32_t b);
/* draw j of (seed, image_index, slot): DESIGN.md O1 counter layout. */
double albref_draw(uint64_t seed, uint64_t image_index, int32_t slot, int32_t j);

/* round_half_up + clamp to [0,255]. */
uint8_t albref_clip_round(double v);
/* reflect-101 index (periodic extension R7). */
int32_t albref_reflect101(int32_t i, int32_t n);

/* GridDistortion axis map (reading R31): source coordinate src[x] of every
 * destination index x in [0, L) for step factors f[0..n] (f[n] is drawn but
 * unused).  Returns ALBREF_E_RANGE for n outside [1, 32] or a factor <= 0. */
int albref_grid_axis(int32_t L, int32_t n, const double* f, double* src);

/* ElasticTransform (reading R32).  Normalised truncated Gaussian of std sigma:
 * w[0..2r], r = ceil(3 sigma); returns r (w must hold 2*48+1 entries), or
 * ALBREF_E_RANGE for sigma outside (0, 16]. */
int albref_gauss_kernel(double sigma, double* w);
/* Displacement planes dx, dy [h][w] of slot `slot` of image `image_index`:
 * raw u, v ~ U(-1, 1) (draws 1 + y w + x, then 1 + h w + y w + x), blurred
 * x then y with w[] and reflect-101 (acc = acc + w x, ascending k), times alpha. */
int albref_elastic_field(int32_t h, int32_t w, double alpha, double sigma, uint64_t seed,
                         uint64_t image_index, int32_t slot, double* dx, double* dy);

/* hexcone colour model, double precision. */
void albref_rgb_to_hsv(double r, double g, double b, double* h, double* s, double* v);
void albref_hsv_to_rgb(double h, double s, double v, double* r, double* g, double* b);

/* Per-image LUT of a LUT-type op, params as drawn (O8).  lut is
 * [3][256] (channel-major).  Returns ALBREF_E_UNSUPPORTED for non-LUT kinds. */
int albref_build_lut(int32_t kind, const double* params, uint8_t* lut);
/* Equalize LUT for one channel (reading R15), hist[256] with N = sum. */
int albref_equalize_lut(const int64_t* hist, uint8_t* lut);

/* Output dims of the pipeline for an h x w input. */
int albref_output_shape(const albref_op* ops, int32_t n_ops, int32_t in_h, int32_t in_w,
                        int32_t* out_h, int32_t* out_w);

/* Params of every slot for one image: params[n_ops][8], fired[n_ops].  The
 * dims each slot sees are tracked through the pipeline (RandomCrop draws
 * depend on the current image size). */
int albref_sample_params(const albref_op* ops, int32_t n_ops, uint64_t seed,
                         uint64_t image_index, int32_t in_h, int32_t in_w,
                         double* params, uint8_t* fired);

/* Apply the pipeline to one sample (SPEC.md:482-490 with DESIGN.md O14).
 *   img [h][w][channels]; mask [h][w] or NULL; boxes [n_boxes][4] or NULL.
 *   Outputs: img_out [oh][ow][channels] (ignored when the pipeline ends in
 *   Normalize, then nchw_out [3][oh][ow] float32 is written); mask_out [oh][ow];
 *   boxes_out/labels_out capacity n_boxes, *n_boxes_out = kept count.
 *   The caller sizes outputs with albref_output_shape. */
int albref_apply(const albref_op* ops, int32_t n_ops, uint64_t seed, uint64_t image_index,
                 const uint8_t* img, int32_t h, int32_t w, int32_t channels,
                 const uint8_t* mask,
                 const float* boxes, const int32_t* labels, int32_t n_boxes,
                 float min_visibility,
                 uint8_t* img_out, float* nchw_out, uint8_t* mask_out,
                 float* boxes_out, int32_t* labels_out, int32_t* n_boxes_out);

/* Nearest-tie candidate sets (SURVEY.md §8(c) tolerance table "Mask nearest",
 * reading R20): the same computation as albref_apply (no boxes; its image /
 * mask / nchw outputs are identical), plus for every output pixel the set of
 * values an implementation may produce when a nearest sample's source
 * coordinate is within ALBREF_TIE_BAND px of a .5 rounding tie (either
 * neighbour accepted).  Sets follow the pixels through exact geometric ops
 * and through pointwise ops; a bilinear sample resets the image set to its
 * own value.  cand_img [oh][ow][ALBREF_MAX_CAND][channels], cand_img_n
 * [oh][ow] (member count; 0 = more than ALBREF_MAX_CAND members: any value),
 * cand_mask [oh][ow][ALBREF_MAX_CAND] / cand_mask_n [oh][ow] (mask given). */
#define ALBREF_MAX_CAND 8
#define ALBREF_TIE_BAND 1e-4
int albref_apply_cand(const albref_op* ops, int32_t n_ops, uint64_t seed, uint64_t image_index,
                      const uint8_t* img, int32_t h, int32_t w, int32_t channels,
                      const uint8_t* mask, uint8_t* img_out, float* nchw_out, uint8_t* mask_out,
                      uint8_t* cand_img, uint8_t* cand_img_n, uint8_t* cand_mask,
                      uint8_t* cand_mask_n);

/* Synthetic-input generator recipe is NOT here (synth/ owns it). */

#ifdef __cplusplus
}
#endif
#endif
