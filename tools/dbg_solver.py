import sys, math, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1606_07652_b200 as B
from paper_1606_07652_b200 import inputs as I, solver as S
x = I.generate_quasiuniform(512, 1, 300, 0.4, lo=(0.0, 0.0), hi=(32.0, 1.0))
ps = B.PointSet(1, x, B.BoundingBox((0.0, 0.0, 0.0), (32.0, 1.0, 1.0)))
k = B.parse_kernel_spec("gaussian:c=256")
v = np.random.default_rng(0).standard_normal(512)
d = B.direct_matvec(k, ps, v).values
for lvl in (4, 5):
    pl = B.Plan(ps, lvl, k, 203.0, 2112)
    f = pl.execute(v).values
    print('level', lvl, 'rel err vs direct', np.abs(f-d).max()/np.abs(d).max())
from oracle import pyoracle as po
ov, st, _ = po.mlfmm(x, v, "gaussian:c=256", 203.0, 2112, 4, lo=[0.0], hi=[32.0])
print('oracle vs direct', np.abs(ov-d).max()/np.abs(d).max(), 'gpu vs oracle', np.abs(B.Plan(ps, 4, k, 203.0, 2112).execute(v).values-ov).max()/np.abs(ov).max())
rhs = np.sin(math.pi * x[:, 0] / 32.0)
for be in S.Backend:
    try:
        lam, st = S.solve_interpolation(S.InterpolationProblem(k, ps, rhs, be, tol=1e-12, sigma=203.0, m_per_dim=2112))
        print(be, st)
    except Exception as e:
        print(be, 'ERR', e, getattr(e, 'achieved', None))
