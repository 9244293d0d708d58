"""Precision experiment (design input, not a test): run the oracle's IK-Beam with
float32 arithmetic and a per-lane float32 Cholesky, and compare with float64.
Usage: PYTHONPATH=. python tools/fp32_oracle_sim.py"""
import numpy as np, time
from oracle import ik_oracle as o
R = "paper_2505_03728_b200/robots/"
ch = o.load_chain_files(R+"arm7.urdf", R+"arm7.sidecar.json")
N=300
tq, tt, _ = o.reachable_targets(ch, 8, N, 77)
seeds = o.sample_seeds(ch, 64, 77)
res64 = o.ik_beam(ch, 8, tq, tt, seeds)
fails=[0,0]
class Chol(o.LaneEngine):
    def _solve(self, h, g):
        n = h.shape[-1]; B=h.shape[0]
        L = np.zeros_like(h); ok = np.ones(B, bool)
        for j in range(n):
            s = h[:, j, j] - np.sum(L[:, j, :j]**2, axis=-1)
            ok &= s > 0
            d = np.sqrt(np.where(s > 0, s, 1).astype(h.dtype))
            L[:, j, j] = d
            for i in range(j+1, n):
                L[:, i, j] = (h[:, i, j] - np.sum(L[:, i, :j]*L[:, j, :j], axis=-1)) / d
        y = np.zeros_like(g)
        for i in range(n):
            y[:, i] = (g[:, i] - np.sum(L[:, i, :i]*y[:, :i], axis=-1)) / L[:, i, i]
        x = np.zeros_like(g)
        for i in reversed(range(n)):
            x[:, i] = (y[:, i] - np.sum(L[:, i+1:, i]*x[:, i+1:], axis=-1)) / L[:, i, i]
        fails[0] += (~ok).sum(); fails[1] += B
        return -x, ok
def stats(name, r):
    print(f"{name:8s} succ {r.success.mean()*100:.2f}% pos p50 {np.percentile(r.pos_err,50):.2e} p98 {np.percentile(r.pos_err,98):.2e} rot p50 {np.percentile(r.rot_err,50):.2e} p98 {np.percentile(r.rot_err,98):.2e} cost p50 {np.percentile(r.cost,50):.3e}")
stats("fp64", res64)
o.LaneEngine = Chol
resc = o.ik_beam(ch, 8, tq, tt, seeds, dtype=np.float32)
stats("chol32", resc); print("fails", fails)
rel = np.abs(resc.hist - res64.hist)/ (res64.hist)
print("p50", np.percentile(rel,50,axis=0).round(6)); print("p90", np.percentile(rel,90,axis=0).round(6))
print("final cost ratio", np.percentile(resc.cost/res64.cost,[50,90,99,100]))
