import os
import sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_05061_b200 as S, oracle as O
rng = np.random.default_rng(6)
A = rng.integers(0, 16, size=(20, 24, 26)).astype(np.float32)
B = np.clip(np.round(0.6 * A + rng.integers(-3, 4, size=A.shape)), 0, 15).astype(np.float32)
A[0, 0, :2] = (0, 15); B[0, 0, :2] = (0, 15)
g = S.Srwcr(A, B, (1, 1, 1), 16, (0, 0, 0), (5, 5, 5), inputs_normalized=True)
D, _ = g.eval(np.zeros(g.params_shape))
a, b = A.ravel().astype(np.float64), B.ravel().astype(np.float64)
within = sum((a == k).mean() * b[a == k].var() for k in np.unique(a))
print("gpu", D, "textbook", within / b.var(), "rel", abs(D - within / b.var()) / (within / b.var()))
pb = O.Problem(dims=(26, 24, 20), L=15, delta=(5, 5, 5), kcells=(0, 0, 0))
N, Sm, Q = O.moments(pb, A, B, np.zeros(pb.params_shape))
reg = g.debug_dump("regions").reshape(-1, 6)
sq = g.debug_dump("SQ")
R = N.shape[0]
print("Q_r gpu", sq[N.size:N.size + 4], "oracle", Q.sum(1)[:4])
print("S_r gpu", sq[:N.size].reshape(N.shape).sum(1)[:4], "oracle", Sm.sum(1)[:4])
print("N gpu", g.debug_dump("N").reshape(N.shape).sum(1)[:4], "oracle", N.sum(1)[:4])
print("reg0 gpu", reg[0], "\nstats", g.stats())
