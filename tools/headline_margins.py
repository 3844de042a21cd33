"""Margin survey for tests/test_gpu_headline.py::test_headline_gradients on
trained fields: repeats the test's checks for several training seeds and
prints every quantity the test asserts on, so a rare failure can be traced
to the assertion that sits closest to its bound."""
import os
import sys

import numpy as np

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
sys.path.insert(0, os.path.join(root, "tests"))
sys.path.insert(0, os.path.join(root, "oracle"))
import test_gpu_headline as H  # noqa: E402


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "config1"
    runs = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    for seed in range(runs):
        for ragged in (False, True):
            m = H._model(case)
            H._train_gpu(m, case, 20, seed=99 + 1000 * seed)
            full = H.CASES[case][5]
            B = full - 37 if ragged else full
            X, T = H._batch(case, B, seed=5 + ragged)
            P = m.params
            lg = m.gradients(X, T, H.CASES[case][3])
            G = m.grads
            lo, ref, emu, cache = H._oracle_grads(case, P, m.sizes, X, T)
            t, w, _ = m.sizes
            got = (G[:t], G[t:t + w], G[t + w:])
            row = [f"seed={seed} ragged={int(ragged)} loss_rel={abs(lg - lo) / abs(lo):.2e}"]
            dset = np.flatnonzero((got[0] != 0) != (ref[0] != 0))
            row.append(f"set_diff={dset.size}")
            if dset.size:
                row.append(f"set_vals got={got[0][dset[:4]]} ref={ref[0][dset[:4]]} emu={emu[0][dset[:4]]} "
                           f"max={np.abs(ref[0]).max():.2e}")
                # which samples touch the differing rows, and their kernel / oracle residuals
                grid = H.CASES[case][0]
                specs = H.O.level_resolutions(H._ocfg(grid))
                F = grid["features"]
                rows_d = set((dset // F).tolist())
                smp = set()
                for l in range(grid["levels"]):
                    r = specs[l].row_offset + cache.rows[l].astype(np.int64)   # [B, 2^d]
                    hit = np.isin(r, list(rows_d)).any(axis=1)
                    smp.update(np.flatnonzero(hit).tolist())
                smp = sorted(smp)[:6]
                pg = m.evaluate(X[smp]).ravel()
                row.append(f"samples={smp} gpu_pred-t={(pg - T[smp].ravel()).tolist()}")
            for name, a, r, e in zip(("tab", "W", "b"), got, ref, emu):
                big = np.abs(r) > 1e-2 * np.abs(r).max()
                dis = int(np.sum(np.sign(a[big]) != np.sign(r[big])))
                dis_e = int(np.sum(np.sign(e[big]) != np.sign(r[big])))
                row.append(f"{name}: emu={H._rel(a, e):.1e} ref={H._rel(a, r):.1e} er={H._rel(e, r):.1e} "
                           f"sign_dis={dis}/{int(big.sum())} emu_dis={dis_e}")
            print(" | ".join(row), flush=True)


if __name__ == "__main__":
    main()
