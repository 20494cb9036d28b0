"""Golden .cngp files and decodes from the REAL reference (model_io.py).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_cngp.py

Builds a few models with the reference (random-perturbed tables, baked from
random confidences so every probe offset occurs), serializes them with the
reference's ``serialize`` and records, per model: the file bytes, the header
fields, the unpacked baked offsets, and the reference's ``decode_pixels`` of
fixed queries after a ``deserialize`` round trip.  Also the FORMAT.md worked
example (87 bytes).  Output: cngp_files.npz next to this script.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import ensure_reference  # noqa: E402

CONFIGS = {
    # name: HyperParams kwargs, image (width, height)
    "np4": (dict(n_f=2**10, n_c=2**12, n_p=4, n_max=512), (64, 48)),
    "np16": (dict(n_f=2**10, n_c=2**10, n_p=16, n_max=1024), (0, 0)),
    "np8_d3": (dict(d=3, n_f=2**8, n_c=2**10, n_p=8, n_max=256, out_dim=1), (0, 0)),
    "np2_sig_f4": (dict(n_f=2**8, n_c=2**9, n_p=2, n_levels=6, n_max=128, feature_dim=4,
                        n_neurons=32, out_sigmoid=True), (17, 9)),
    "np1": (dict(n_f=2**10, n_c=2**10, n_p=1, n_max=512), (0, 0)),
}


def main():
    ensure_reference()
    from probegrid.model import HyperParams, init_model
    from probegrid.model_io import decode_pixels, deserialize, serialize, to_inference

    out = {}
    for name, (kw, (w, h)) in CONFIGS.items():
        hyper = HyperParams(**kw)
        m = init_model(hyper, seed=3)
        rng = np.random.default_rng(7)
        for lv in m.levels:
            lv.features.values[:] = (rng.standard_normal(lv.features.values.shape) * 0.3).astype(np.float32)
            if lv.conf is not None:
                lv.conf.values[:] = rng.standard_normal(lv.conf.values.shape).astype(np.float32)
                lv.baked.entries[:] = np.argmax(lv.conf.values, axis=1).astype(np.uint8)
        for b in m.mlp.biases:
            b[:] = (rng.standard_normal(b.shape) * 0.1).astype(np.float32)
        raw = serialize(to_inference(m, width=w, height=h))
        inf = deserialize(raw)
        q = np.random.default_rng(11).random((2000, hyper.d), dtype=np.float32)
        q[0] = 0.0
        q[1] = 1.0
        out[f"{name}_file"] = np.frombuffer(raw, np.uint8)
        out[f"{name}_xs"] = q
        out[f"{name}_decode"] = decode_pixels(inf, q)
        out[f"{name}_baked"] = np.array([b for b in inf.baked if b is not None] or
                                        np.zeros((0, hyper.n_c), np.uint8))
        out[f"{name}_kw"] = np.array(sorted((k, str(v)) for k, v in kw.items()))
    # FORMAT.md worked example: built through the reference API, 87 bytes
    hyper = HyperParams(d=2, n_levels=1, feature_dim=1, n_min=2, n_max=2, n_f=4, n_c=8, n_p=2,
                        n_neurons=2, n_hidden_layers=1, out_dim=3)
    m = init_model(hyper, seed=0)
    m.levels[0].features.values[:, 0] = [0.5, 1.0, -2.0, 0.25]
    m.levels[0].baked.entries[:] = [1, 0, 1, 1, 0, 0, 1, 0]
    for wgt, b in zip(m.mlp.weights, m.mlp.biases):
        wgt[:] = 0.5
        b[:] = -1.0
    ex = serialize(to_inference(m, width=3, height=2))
    assert len(ex) == 87, len(ex)
    out["format_example_file"] = np.frombuffer(ex, np.uint8)
    # trainer.select_hyperparams (size-budgeted configurations)
    from probegrid.model_io import size_report
    from probegrid.trainer import select_hyperparams
    floor = size_report(HyperParams(n_f=2**6, n_c=2**10, n_p=2**1)).total_bytes
    targets = [floor, floor + 1, 25_000, 60_000, 150_000, 300_000, 1_000_000, 5_000_000, 10**8]
    sel = []
    for t in targets:
        h = select_hyperparams(t)
        sel.append([t, h.n_f, h.n_c, h.n_p, size_report(h).total_bytes])
    out["select_hyperparams"] = np.array(sel, np.int64)
    np.savez_compressed(os.path.join(HERE, "cngp_files.npz"), **out)
    print("cngp_files.npz", os.path.getsize(os.path.join(HERE, "cngp_files.npz")))


if __name__ == "__main__":
    main()
