"""Generate golden vectors from the REAL reference package (probegrid).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to /tmp/refbuild (read-only source), builds the
reference's Cython core there with the reference's own setup.py, imports
``probegrid`` from that copy and records inputs + outputs of the hot-path
functions into small .npz fixtures next to this script.  The fixtures pin
the CPU oracle (oracle/oracle.py) in tests/test_oracle.py; the GPU parity
tests then compare the CUDA path against the oracle.
"""

import hashlib
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg"
BUILD = os.environ.get("PROBEGRID_REFBUILD", "/tmp/refbuild")


def ensure_reference():
    so_glob = os.path.join(BUILD, "src", "probegrid", "backends")
    built = os.path.isdir(so_glob) and any(f.startswith("_core") and f.endswith(".so")
                                           for f in os.listdir(so_glob))
    if not built:
        shutil.rmtree(BUILD, ignore_errors=True)
        shutil.copytree(REF_PKG, BUILD)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=BUILD,
                       check=True, stdout=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(BUILD, "src"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def geometry(seed, b, d, dtype, res_list):
    """Random points plus the reference test's edges (test_backends.py:19-25)
    plus near-vertex points k/res nudged by a few ulps (SURVEY 7.4 hazard 1)."""
    rng = np.random.default_rng(seed)
    xs = rng.random((b, d)).astype(dtype)
    xs[0] = 0.0
    xs[1] = 1.0
    xs[2, 0] = 1.0
    extra = []
    for res in res_list:
        ks = rng.integers(1, res, size=24)
        for k in ks:
            v = dtype(k) / dtype(res)
            for n in (-2, -1, 0, 1, 2):
                x = v
                step = np.inf if n > 0 else -np.inf
                for _ in range(abs(n)):
                    x = np.nextafter(x, dtype(step))
                if 0 <= x <= 1:
                    p = rng.random(d).astype(dtype)
                    p[rng.integers(0, d)] = x
                    extra.append(p)
    return np.concatenate([xs, np.array(extra, dtype=dtype)]).astype(dtype)


def main():
    ensure_reference()
    from probegrid.backends import cython_backend as cy
    from probegrid.backends import numpy_backend as npb
    from probegrid.indexing import AUX_PRIMES, PRIMARY_PRIMES
    from probegrid.mlp import mlp_backward, mlp_forward, mlp_init
    from probegrid.model import HyperParams, init_model
    from probegrid.model_io import decode_pixels, to_inference
    from probegrid.trainer import TrainConfig, TrainState

    out = {}
    # ---- forward kernels (test_backends.py:28-64 shapes + hazard points) ----
    for dt in (np.float32, np.float64):
        tag = np.dtype(dt).name
        for d in (2, 3):
            rng = np.random.default_rng(100 + d)
            xs = geometry(d, 257, d, dt, [8, 21, 33, 322])
            dense_feats = rng.standard_normal((9 ** d, 2)).astype(dt)
            feats = rng.standard_normal((64, 2)).astype(dt)
            baked = rng.integers(0, 4, size=32).astype(np.uint8)
            k = f"{tag}_d{d}"
            out[f"fwd_{k}_xs"] = xs
            out[f"fwd_{k}_dense_feats"] = dense_feats
            out[f"fwd_{k}_feats"] = feats
            out[f"fwd_{k}_baked"] = baked
            o, idx, w = cy.dense_fwd(xs, 8, dense_feats)
            out.update({f"fwd_{k}_dense_out": o, f"fwd_{k}_dense_idx": idx, f"fwd_{k}_dense_w": w})
            o, idx, w = cy.hashed_fwd(xs, 33, 64, feats, PRIMARY_PRIMES)
            out.update({f"fwd_{k}_hashed_out": o, f"fwd_{k}_hashed_idx": idx,
                        f"fwd_{k}_hashed_w": w})
            o, base, row, w = cy.probed_fwd(xs, 21, 64, 32, 2, feats, baked, PRIMARY_PRIMES,
                                            AUX_PRIMES)
            out.update({f"fwd_{k}_probed_out": o, f"fwd_{k}_probed_base": base,
                        f"fwd_{k}_probed_row": row, f"fwd_{k}_probed_w": w})
            # hazard: res 322 probed, bigger tables
            feats2 = rng.standard_normal((4096, 2)).astype(dt)
            baked2 = rng.integers(0, 4, size=1 << 14).astype(np.uint8)
            out[f"fwd_{k}_feats2"] = feats2
            out[f"fwd_{k}_baked2"] = baked2
            o, base, row, w = cy.probed_fwd(xs, 322, 4096, 1 << 14, 2, feats2, baked2,
                                            PRIMARY_PRIMES, AUX_PRIMES)
            out.update({f"fwd_{k}_p322_out": o, f"fwd_{k}_p322_base": base,
                        f"fwd_{k}_p322_row": row, f"fwd_{k}_p322_w": w})
    np.savez_compressed(os.path.join(HERE, "fwd_kernels.npz"), **out)

    # ---- backward kernels (test_backends.py:67-106) ----
    out = {}
    for dt in (np.float32, np.float64):
        tag = np.dtype(dt).name
        for F in (2, 4):
            rng = np.random.default_rng(5 + F)
            n_f, n_c, n_p = 64, 32, 4
            up = rng.standard_normal((257, F)).astype(dt)
            idx = rng.integers(0, 64, size=(257, 4)).astype(np.int32)
            base = (rng.integers(0, n_f // n_p, size=(257, 4)) * n_p).astype(np.int32)
            row = rng.integers(0, n_c, size=(257, 4)).astype(np.int32)
            wgt = rng.random((257, 4)).astype(dt)
            conf = rng.standard_normal((n_c, n_p)).astype(dt)
            feats = rng.standard_normal((n_f, F)).astype(dt)
            gi = np.zeros((n_f, F), dt)
            cy.indexed_bwd(up, idx, wgt, gi)
            rows_u, inv = cy.dedup_rows(row, n_c)
            smu = npb.softmax_rows(conf[rows_u])
            gf = np.zeros((n_f, F), dt)
            gcu = np.zeros_like(smu)
            cy.probed_bwd(up, base, inv, wgt, smu, feats, gf, gcu)
            k = f"{tag}_F{F}"
            out.update({f"bwd_{k}_up": up, f"bwd_{k}_idx": idx, f"bwd_{k}_base": base,
                        f"bwd_{k}_row": row, f"bwd_{k}_w": wgt, f"bwd_{k}_conf": conf,
                        f"bwd_{k}_feats": feats, f"bwd_{k}_gidx": gi, f"bwd_{k}_rows_u": rows_u,
                        f"bwd_{k}_inv": inv, f"bwd_{k}_smu": smu, f"bwd_{k}_gfeat": gf,
                        f"bwd_{k}_gconf_u": gcu})
        # adam_rebake_rows (test_backends.py:108-136)
        rng = np.random.default_rng(6)
        conf = rng.standard_normal((16, 4)).astype(dt)
        m = (rng.standard_normal((16, 4)) * 0.01).astype(dt)
        v = (rng.random((16, 4)) * 0.01).astype(dt)
        baked = np.argmax(conf, axis=1).astype(np.uint8)
        rows_u = np.array([3, 7, 1, 12], np.int32)
        g = rng.standard_normal((4, 4)).astype(dt)
        # ties: row 5 all equal after update is unlikely; add an explicit tie row
        conf[9] = 0.5
        rows_u = np.array([3, 7, 1, 12, 9], np.int32)
        g = np.concatenate([g, np.zeros((1, 4), dt)])
        out.update({f"adam_{tag}_conf": conf.copy(), f"adam_{tag}_m": m.copy(),
                    f"adam_{tag}_v": v.copy(), f"adam_{tag}_baked": baked.copy(),
                    f"adam_{tag}_rows_u": rows_u, f"adam_{tag}_g": g})
        cy.adam_rebake_rows(conf, m, v, baked, rows_u, g, 5, 1e-2, 0.9, 0.99, 1e-15)
        out.update({f"adam_{tag}_conf_out": conf, f"adam_{tag}_m_out": m,
                    f"adam_{tag}_v_out": v, f"adam_{tag}_baked_out": baked})
    np.savez_compressed(os.path.join(HERE, "bwd_kernels.npz"), **out)

    # ---- MLP (test_backends.py:139-171, test_mlp.py) ----
    out = {}
    rng = np.random.default_rng(11)
    p = mlp_init(rng, [32, 64, 64, 3], np.float32)
    xs = rng.standard_normal((96, 32)).astype(np.float32)
    out["mlp_W"] = np.array(p.weights, dtype=object)
    for i, (w, b) in enumerate(zip(p.weights, p.biases)):
        p.biases[i][:] = rng.standard_normal(b.shape).astype(np.float32) * 0.1
        out[f"mlp_W{i}"] = w
        out[f"mlp_b{i}"] = p.biases[i]
    del out["mlp_W"]
    out["mlp_x"] = xs
    out["mlp_rows"] = cy.mlp_infer_rows(xs, p.weights, p.biases)
    out["mlp_rows_sig"] = cy.mlp_infer_rows(xs, p.weights, p.biases, out_sigmoid=True)
    o, cache = mlp_forward(p, xs)
    up = rng.standard_normal(o.shape).astype(np.float32)
    dx = mlp_backward(p, cache, up)
    out["mlp_fwd"] = o
    out["mlp_up"] = up
    out["mlp_dx"] = dx
    for i in range(3):
        out[f"mlp_Wg{i}"] = p.weight_grads[i]
        out[f"mlp_bg{i}"] = p.bias_grads[i]
    np.savez_compressed(os.path.join(HERE, "mlp.npz"), **out)

    # ---- init + training trajectories + decode ----
    out = {}
    small = dict(n_f=32, n_c=64, n_p=4, n_levels=3, n_min=4, n_max=16, n_neurons=8)
    out["small_hyper"] = np.array(list(small.items()), dtype=object).astype(str)
    m = init_model(HyperParams(**small), seed=0)
    for i, lv in enumerate(m.levels):
        out[f"small_init_feats{i}"] = lv.features.values
        if lv.conf is not None:
            out[f"small_init_conf{i}"] = lv.conf.values
            out[f"small_init_baked{i}"] = lv.baked.entries
    for i, w in enumerate(m.mlp.weights):
        out[f"small_init_W{i}"] = w
    # C1 init fingerprints
    c1 = HyperParams(n_f=2**12, n_c=2**14, n_p=4)
    m1 = init_model(c1, seed=0)
    fp = []
    for i, lv in enumerate(m1.levels):
        fp.append(f"feats{i}:{sha(lv.features.values)}")
        if lv.conf is not None:
            fp.append(f"conf{i}:{sha(lv.conf.values)}")
            fp.append(f"baked{i}:{sha(lv.baked.entries)}")
    for i, w in enumerate(m1.mlp.weights):
        fp.append(f"W{i}:{sha(w)}")
    out["c1_init_sha"] = np.array(fp)
    out["c1_levels"] = np.array([[lv.spec.resolution, lv.spec.mode.value == "dense"]
                                 for lv in m1.levels])
    # trajectories: tiny config (full params) and C1 (losses + hashes)
    img = np.random.default_rng(9).random((16, 16, 3)).astype(np.float32)
    st = TrainState(init_model(HyperParams(**small), seed=0), img,
                    TrainConfig(steps=30, batch_size=128, seed=0))
    out["small_img"] = img
    out["small_losses"] = np.array([st.step() for _ in range(30)])
    for i, lv in enumerate(st.model.levels):
        out[f"small_final_feats{i}"] = lv.features.values
        if lv.conf is not None:
            out[f"small_final_conf{i}"] = lv.conf.values
            out[f"small_final_baked{i}"] = lv.baked.entries
    for i, (w, b) in enumerate(zip(st.model.mlp.weights, st.model.mlp.biases)):
        out[f"small_final_W{i}"] = w
        out[f"small_final_b{i}"] = b

    yy, xx = np.mgrid[0:256, 0:256]
    u = (xx + 0.5) / 256
    v = (yy + 0.5) / 256
    smooth = np.stack([0.5 + 0.5 * np.sin(6 * np.pi * u) * np.cos(4 * np.pi * v), u,
                       0.5 + 0.25 * np.sin(10 * np.pi * (u + v))], -1).astype(np.float32)
    st = TrainState(init_model(c1, seed=0), smooth, TrainConfig(steps=5, batch_size=8192, seed=0))
    out["c1_losses"] = np.array([st.step() for _ in range(5)])
    fp = []
    for i, lv in enumerate(st.model.levels):
        fp.append(f"feats{i}:{sha(lv.features.values)}")
        if lv.conf is not None:
            fp.append(f"baked{i}:{sha(lv.baked.entries)}")
    out["c1_step5_sha"] = np.array(fp)
    out["c1_step5_feat_sum"] = np.array([float(np.sum(lv.features.values.astype(np.float64)))
                                         for lv in st.model.levels])
    inf = to_inference(st.model)
    q = np.random.default_rng(1234).random((3000, 2), dtype=np.float32)
    q[0] = 0.0
    q[1] = 1.0
    out["c1_decode_xs"] = q
    out["c1_decode_out"] = decode_pixels(inf, q)
    np.savez_compressed(os.path.join(HERE, "model_traj.npz"), **out)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
