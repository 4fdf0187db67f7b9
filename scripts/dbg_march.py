import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from helpers import oracle_aligned, soa
from paper_2403_01004_b200 import configs, operators
for n in [(24, 24, 48), (16, 16, 64), (16, 8, 32), (12, 8, 32)]:
    w = configs.c3(n=n)
    cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
    T = operators.Field(w.grid, w.fields["T"])
    op = operators.DiffusionOperator.aligned(cfg, T)
    F = op.apply(T).values[..., 0]
    oop = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"])
    Fo = oop.apply(soa(w.fields["T"][..., None]))[0]
    bad = np.argwhere(F != Fo)
    print(n, "nbad", len(bad), "max rel", np.max(np.abs(F - Fo)) / np.max(np.abs(Fo)))
    if len(bad):
        print(" i values", np.unique(bad[:, 0])[:20], " j", np.unique(bad[:, 1])[:20], " k", np.unique(bad[:, 2])[:40])
        for b in bad[:5]:
            print("  ", tuple(b), F[tuple(b)], Fo[tuple(b)])
