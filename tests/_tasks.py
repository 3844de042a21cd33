"""Test-side restatement of the reference's fit_image loop (tasks.cpp:49-128).

Drives any model exposing ``train_step(X, target, loss_kind, step)`` and
``evaluate(X)`` (the oracle's Field or the GPU FieldModel) with the reference's
exact batch stream: Pcg32(seed, 1).next_below(w*h) per sample (tasks.cpp:112-120).
"""
import numpy as np

import oracle as O


def eval_grid(w: int, h: int, seed: int):   # tasks.cpp:74-93
    n = w * h
    if n <= (1 << 20):
        pix = np.arange(n)
    else:
        r = O.Pcg32(seed, 7)
        pix = np.array([r.next_below(n) for _ in range(1 << 16)])
    X = np.stack([((pix % w) + 0.5) / w, ((pix // w) + 0.5) / h], axis=1).astype(np.float32)
    # float arithmetic as in the reference: (float(p % w) + 0.5f) / float(w)
    X[:, 0] = ((pix % w).astype(np.float32) + np.float32(0.5)) / np.float32(w)
    X[:, 1] = ((pix // w).astype(np.float32) + np.float32(0.5)) / np.float32(h)
    return X, pix


def evaluate_chunked(model, X, chunk=1 << 16):   # tasks.cpp:34-45
    if X.shape[0] <= chunk:
        return model.evaluate(X)
    return np.concatenate([model.evaluate(X[c:c + chunk]) for c in range(0, X.shape[0], chunk)])


def fit_image(model, rgb, w, h, seed, batch, total_steps, log_interval):
    """Returns report rows (step, loss, psnr). ``model`` must already be init(seed)'d
    with the default schedule for total_steps."""
    ex, pix = eval_grid(w, h, seed)
    et = rgb[pix]
    rows = []
    pred = evaluate_chunked(model, ex)
    rows.append((0, float(((pred - et) ** 2).mean()), O.psnr(pred, et)))
    rng = O.Pcg32(seed, 1)
    for step in range(1, total_steps + 1):
        X, t = rng.image_batch(rgb, w, h, batch)
        loss = model.train_step(X, t, O.LOSS_L2, step)
        if not np.isfinite(loss):
            raise RuntimeError(f"fit_image: non-finite loss at step {step}")
        if step % log_interval == 0 or step == total_steps:
            pred = evaluate_chunked(model, ex)
            rows.append((step, float(loss), O.psnr(pred, et)))
    return rows
