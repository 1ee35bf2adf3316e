import sys, os, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1906_00142_b200 import fit as G, formats as F
from oracle import o3_fit as O3
rng = np.random.default_rng(1906)
m = 1000000
D = rng.integers(64, 65537, m).astype(float)
cfg = np.array(F.integer_configs(), dtype=float)[rng.integers(0, 7262, m)][:, :2]
X = np.ascontiguousarray(np.column_stack([D, cfg]))
spec = F.load_kernel_spec("/root/repo/data/polybench/gemm.kernel.json")
for name in F.REQUIRED_METRICS:
    y = O3.eval_ratfunc(spec.ground_truth[name], X) * (1 + rng.uniform(-0.01, 0.01, m))
    y = np.ascontiguousarray(y)
    res = []
    for rep in range(3):
        f, r = G.fit_rational(X, y, spec.variables, [2,2,2], [1,1,1])
        res.append(np.array(f.num.coeffs + f.den.coeffs))
    same = all(np.array_equal(res[0], q) for q in res[1:])
    print(name, "deterministic" if same else "DIFFERS", r.safeguard, np.max(np.abs(res[0]-res[1])))
