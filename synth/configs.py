"""Workload definitions of BASELINE.json configs 1-5 as plain op-spec dicts.

An op spec is a dict: kind (DESIGN.md op names), p, lo/hi parameter ranges
(param j = lo[j] + (hi[j]-lo[j])*u), size=(w, h), side=(min, max),
origin=(x, y), interp, border, fill, mask_fill, mean, std.  Both the CUDA
binding and the oracle wrapper convert these dicts into their own structs.
No arithmetic of the method lives here.
"""

IMAGENET_MEAN = (0.485, 0.456, 0.406)   # reading R16
IMAGENET_STD = (0.229, 0.224, 0.225)


def op(kind, **kw):
    d = {"kind": kind, "p": 1.0}
    d.update(kw)
    return d


# cfg1 (BASELINE.json configs[0]): HFlip, VFlip, Brightness(+-0.2), Gamma(80-120)
CFG1_OPS = {
    "HorizontalFlip": [op("HorizontalFlip")],
    "VerticalFlip": [op("VerticalFlip")],
    "Brightness": [op("Brightness", lo=[0.8], hi=[1.2])],
    "Gamma": [op("Gamma", lo=[0.8], hi=[1.2])],
}
CFG1_COMPOSE = [op("HorizontalFlip", p=0.5), op("VerticalFlip", p=0.5),
                op("Brightness", p=0.5, lo=[0.8], hi=[1.2]),
                op("Gamma", p=0.5, lo=[0.8], hi=[1.2])]

WARP = dict(interp="bilinear", border="reflect_101")
SSR_LO = [-0.0625, -0.0625, 0.9, -45.0]
SSR_HI = [0.0625, 0.0625, 1.1, 45.0]

# cfg2 (BASELINE.json configs[1]): the 16 single transforms, p = 1 (R4/R5/R11/R13)
CFG2_MENU = {
    "HorizontalFlip": [op("HorizontalFlip")],
    "VerticalFlip": [op("VerticalFlip")],
    "Rotate": [op("Rotate", lo=[-90.0], hi=[90.0], **WARP)],
    "ShiftScaleRotate": [op("ShiftScaleRotate", lo=SSR_LO, hi=SSR_HI, **WARP)],
    "Brightness": [op("Brightness", lo=[0.8], hi=[1.2])],
    "Contrast": [op("Contrast", lo=[0.8], hi=[1.2])],
    "BrightnessContrast": [op("BrightnessContrast", lo=[0.8, 0.8], hi=[1.2, 1.2])],
    "ShiftRGB": [op("ShiftRGB", lo=[-20.0] * 3, hi=[20.0] * 3)],
    "ShiftHSV": [op("ShiftHSV", lo=[-20.0, -0.1, -0.1], hi=[20.0, 0.1, 0.1])],
    "Gamma": [op("Gamma", lo=[0.8], hi=[1.2])],
    "Grayscale": [op("Grayscale")],
    "RandomCrop64": [op("RandomCrop", size=(64, 64))],
    "PadToSize512": [op("PadToSize", size=(512, 512))],
    "Resize512": [op("Resize", size=(512, 512), interp="bilinear")],
    "RandomSizedCrop64-512": [op("RandomSizedCrop", side=(64, 512), size=(512, 512),
                                 interp="bilinear")],
    "Equalize": [op("Equalize")],
}

# cfg3 (configs[2]): 512x512 + mask, Rotate(+-90) / SSR, bilinear, reflect_101
CFG3_OPS = {
    "Rotate": [op("Rotate", lo=[-90.0], hi=[90.0], **WARP)],
    "ShiftScaleRotate": [op("ShiftScaleRotate", lo=SSR_LO, hi=SSR_HI, **WARP)],
}

# cfg4 (configs[3]): RSC(64-375)->Resize 224->HFlip p=.5->ShiftHSV->BC->Normalize
CFG4_OPS = [
    op("RandomSizedCrop", side=(64, 375), size=(224, 224), interp="bilinear"),
    op("Resize", size=(224, 224), interp="bilinear"),
    op("HorizontalFlip", p=0.5),
    op("ShiftHSV", lo=[-20.0, -0.1, -0.1], hi=[20.0, 0.1, 0.1]),
    op("BrightnessContrast", lo=[0.8, 0.8], hi=[1.2, 1.2]),
    op("Normalize", mean=IMAGENET_MEAN, std=IMAGENET_STD),
]

# cfg5 (configs[4]): SSR + RandomCrop 512 + HFlip(p=.5) on image, mask, boxes
CFG5_OPS = [
    op("ShiftScaleRotate", lo=SSR_LO, hi=SSR_HI, **WARP),
    op("RandomCrop", size=(512, 512)),
    op("HorizontalFlip", p=0.5),
]
CFG5_MIN_VISIBILITY = 0.3
CFG5_MAX_BOXES = 50

CONFIGS = {
    1: dict(n=64, size=(256, 256)),
    2: dict(n=2000, size=None),          # ragged, synth.gen.cfg2_sizes
    3: dict(n=256, size=(512, 512)),
    4: dict(n=1024, size=(375, 500)),    # H=375, W=500 (R23)
    5: dict(n=512, size=(1024, 1024)),
}


# next-row transforms measured by tools/copy_probe.py / profile_ops.py on the cfg2 corpus
EXTRA_OPS = {"Rot90k1": [{"kind": "Rotate90", "lo": [1], "hi": [1]}],
             "D4e5": [{"kind": "D4", "lo": [5], "hi": [5]}],
             "D4e2": [{"kind": "D4", "lo": [2], "hi": [2]}],
             "Grid5": [{"kind": "GridDistortion", "lo": [-0.3], "hi": [0.3], "num_steps": 5}],
             "Elastic": [{"kind": "ElasticTransform", "lo": [34.0, 4.0], "hi": [34.0, 4.0], "border": "reflect_101"}],
             "Grid5n": [{"kind": "GridDistortion", "lo": [-0.3], "hi": [0.3], "num_steps": 5, "interp": "nearest"}],
             # SSR whose scale range reaches below 0.9: runs the one-CTA-per-tile affine kernel
             "SSRgen": [op("ShiftScaleRotate", lo=[-0.0625, -0.0625, 0.89, -45.0], hi=SSR_HI, **WARP)]}
