"""Golden-vector dumper: runs the pinned CPU oracle
(oracle/, checked against the reference's own KATs by tests/test_oracle_*.py)
on fixed seeds and writes tests/golden/field_vectors.npz.

Per case it stores the level table, a digest of the initial parameters, the
corner rows and weights, the encoded features, the MLP output, the loss and its
gradient, the MLP and (sparse) table gradients, and the parameters after one
Adam step. The GPU tests (tests/test_gpu_golden.py) read these fixtures
without running the oracle; tests/test_golden_cpu.py checks that the oracle
still reproduces them.

Cases: a small 2-D grid, BASELINE config 1 (2-D image, 3 outputs, L2) and
BASELINE config 2 (3-D SDF, MAPE). Batches are capped (the configs' own batch
sizes are bench workloads) so the file stays small.

    python tools/dump_golden.py            # rewrites tests/golden/field_vectors.npz
"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O   # noqa: E402

CASES = {
    "small": dict(grid=dict(dims=2, levels=8, table_size=1 << 10, features=2, n_min=8, n_max=200, smoothstep=False),
                  n_out=1, sigmoid=False, loss=0, batch=96, seed=7),
    "config1": dict(grid=dict(dims=2, levels=16, table_size=1 << 14, features=2, n_min=16, n_max=1024, smoothstep=False),
                    n_out=3, sigmoid=False, loss=0, batch=128, seed=1337),
    "config2": dict(grid=dict(dims=3, levels=16, table_size=1 << 19, features=2, n_min=16, n_max=2048, smoothstep=False),
                    n_out=1, sigmoid=False, loss=1, batch=64, seed=1337),
}
LR = 1e-2


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def case_vectors(name: str, c: dict) -> dict:
    g = O.GridCfg(**c["grid"])
    mc = O.MlpCfg(g.output_width, 2, 64, c["n_out"], c["sigmoid"])
    f = O.Field(g, mc, O.Hyper(lr=LR))
    f.init(c["seed"])
    P0 = f.params.copy()
    t, w = f.n_tab, f.n_w
    rng = O.Pcg32(c["seed"] + 101, 5)
    B, d = c["batch"], g.dims
    X = rng.floats(B * d).reshape(B, d).astype(np.float32)
    X[:3] = [[0.0] * d, [1.0] * d, [0.5] * d]                 # domain corners and centre
    T = (rng.floats(B * c["n_out"]).reshape(B, c["n_out"]) * 0.6 + 0.2).astype(np.float32)
    Y, cache = O.encode_forward(g, P0[:t], X)
    out = O.mlp_forward(mc, P0[t:t + w], P0[t + w:], Y)
    loss, dpred = O.loss_with_grad(c["loss"], out, T)
    _, gW, gb, dY = O.mlp_forward_backward(mc, P0[t:t + w], P0[t + w:], Y, dpred)
    gt = np.zeros(t, np.float32)
    O.encode_backward(g, cache, dY, gt)
    nz = np.flatnonzero(gt).astype(np.int64)
    step_loss = f.train_step(X, T, c["loss"], 1)
    P1 = f.params.copy()
    specs = O.level_resolutions(g)
    p = f"{name}/"
    return {
        p + "grid": np.array([g.dims, g.levels, g.table_size, g.features, g.n_min, g.n_max, int(g.smoothstep)], np.int64),
        p + "mlp": np.array([c["n_out"], int(c["sigmoid"]), c["loss"], c["seed"]], np.int64),
        p + "resolution": np.array([s.resolution for s in specs], np.int64),
        p + "row_offset": np.array([s.row_offset for s in specs], np.int64),
        p + "params0_sha256": np.array(digest(P0)),
        p + "params0_head": P0[:512].copy(),
        p + "mlp_params0": P0[t:].copy(),
        p + "X": X,
        p + "target": T,
        p + "rows": cache.rows,
        p + "weights": cache.weights.astype(np.float32),
        p + "Y": Y.astype(np.float32),
        p + "out": np.asarray(out, np.float32),
        p + "loss": np.float64(loss),
        p + "dpred": np.asarray(dpred, np.float32),
        p + "grad_mlp": np.concatenate([np.asarray(gW, np.float32).ravel(), np.asarray(gb, np.float32).ravel()]),
        p + "grad_table_index": nz,
        p + "grad_table_value": gt[nz],
        p + "step1_loss": np.float64(step_loss),
        p + "params1_table_touched": P1[:t][nz],
        p + "params1_mlp": P1[t:].copy(),
        p + "params1_untouched_sha256": np.array(digest(np.delete(P1[:t], nz))),
    }


def main() -> None:
    vec = {}
    for name, c in CASES.items():
        vec.update(case_vectors(name, c))
    path = os.path.join(ROOT, "tests", "golden", "field_vectors.npz")
    np.savez_compressed(path, **vec)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.0f} KiB, {len(vec)} arrays)")


if __name__ == "__main__":
    main()
