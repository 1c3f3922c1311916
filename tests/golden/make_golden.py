"""Generate tests/golden/ref_vectors.npz from the UNMODIFIED reference.

Run in the builder container (needs oracle/_ref/liblcnn_ref.so, built from
/root/reference/proj sources by `make -C oracle`).  The resulting fixture is
committed so the GPU box -- which has no /root/reference -- can pin both the
C oracle and the CUDA kernels to the reference's own outputs.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import CHWN, HWCN, NCHW, NHWC, Ref, rng_uniform  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_vectors.npz")


def main():
    v = {}
    seed = 1000
    # transforms: CHWN<->NCHW through the tiled path, other pairs naive
    tshapes = [(3, 5, 7, 2), (48, 3, 5, 5), (96, 5, 7, 3), (1, 3, 4, 4), (64, 3, 9, 11), (7, 2, 3, 5)]
    pairs = [(CHWN, NCHW), (NCHW, CHWN), (NCHW, NHWC), (CHWN, HWCN), (NHWC, HWCN)]
    k = 0
    for shp in tshapes:
        for sl, dl in pairs:
            seed += 1
            x = rng_uniform(seed, int(np.prod(shp)), -100, 100)
            v[f"transform_{k}_in"] = x
            v[f"transform_{k}_meta"] = np.array([*shp, sl, dl], np.int64)
            v[f"transform_{k}_out"] = Ref.transform(x, *shp, sl, dl)
            k += 1
    # pooling: layout kernels, coarsened kernel, fp64 oracle
    pcases = [((4, 3, 13, 13), (3, 3, 2)), ((4, 3, 12, 12), (2, 2, 2)), ((3, 2, 9, 11), (3, 3, 1)),
              ((2, 3, 10, 7), (2, 3, 1)), ((5, 2, 15, 15), (3, 3, 2)), ((1, 1, 3, 11), (3, 3, 2))]
    k = 0
    for shp, (wh, ww, s) in pcases:
        for avg in (0, 1):
            seed += 1
            x = rng_uniform(seed, int(np.prod(shp)), -10, 10)
            for layout in (CHWN, NCHW):
                out, rep = Ref.pool_layout(x, *shp, layout, wh, ww, s, avg)
                v[f"pool_{k}_in"] = x
                v[f"pool_{k}_meta"] = np.array([*shp, layout, wh, ww, s, avg], np.int64)
                v[f"pool_{k}_out"] = out
                v[f"pool_{k}_report"] = np.array(rep, np.uint64)
                v[f"pool_{k}_oracle"] = Ref.pool_oracle(x, *shp, layout, wh, ww, s, avg)
                if layout == CHWN:
                    for fh, fw in ((2, 2), (1, 3), (3, 1), (4, 4)):
                        o2, r2 = Ref.pool_coarsened(x, *shp, layout, wh, ww, s, avg, fh, fw)
                        v[f"pool_{k}_coarse_{fh}x{fw}_out"] = o2
                        v[f"pool_{k}_coarse_{fh}x{fw}_report"] = np.array(r2, np.uint64)
                k += 1
    # softmax: five-pass and fused (incl. the streaming schedule)
    scases = [(1, 1), (3, 7), (16, 10), (8, 1000), (4, 1000), (2, 20000), (5, 4097)]
    for k, (r, c) in enumerate(scases):
        seed += 1
        x = rng_uniform(seed, r * c, -5, 5)
        v[f"softmax_{k}_in"] = x
        v[f"softmax_{k}_meta"] = np.array([r, c], np.int64)
        v[f"softmax_{k}_ref"] = Ref.softmax_reference(x, r, c)[0]
        v[f"softmax_{k}_fused"] = Ref.softmax_fused(x, r, c)[0]
    # convolution (whole-network path): fp64 oracle and the direct kernel
    ccases = [((2, 3, 9, 9), (4, 3, 1, 1)), ((3, 2, 7, 7), (5, 5, 2, 2)), ((2, 4, 11, 11), (6, 3, 2, 0)),
              ((4, 3, 12, 12), (8, 5, 1, 2))]
    for k, ((n, ci, h, w), (co, f, stride, pad)) in enumerate(ccases):
        seed += 1
        x = rng_uniform(seed, n * ci * h * w)
        filt = rng_uniform(seed + 7, co * ci * f * f)
        v[f"conv_{k}_in"] = x
        v[f"conv_{k}_filt"] = filt
        v[f"conv_{k}_meta"] = np.array([n, ci, h, w, co, f, stride, pad], np.int64)
        v[f"conv_{k}_oracle"] = Ref.conv_oracle(x, filt, n, ci, h, w, NCHW, co, f, f, stride, pad)
    np.savez_compressed(OUT, **v)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(v)} arrays)")


if __name__ == "__main__":
    main()
