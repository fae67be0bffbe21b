"""A fitted d = 15 rate matrix (N = 16, V = 1e6, 20 sweeps) as raw float64 for tools/sweep_probe.cu:
    python tools/gen_rate_fixture.py && ./sweep_probe tools/data/rate15.bin"""
import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2401_10068_b200 import model, vb
N = 16
hp = model.default_hyperparams(N)
dd = model.regime(1_000_000, 3, N)
st, _ = vb.vb_fit(dd, hp, max_iter=20)
L = np.ascontiguousarray(st.lam0l_inv, dtype=np.float64)
print(L.shape, np.linalg.eigvalsh(L)[[0, -1]], L[0, :4])
os.makedirs("tools/data", exist_ok=True)
L.tofile("tools/data/rate15.bin")
