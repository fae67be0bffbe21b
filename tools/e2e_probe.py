import time, numpy as np, sys
sys.path.insert(0, '.')
from paper_2401_10068_b200 import _lib, model, vb
V, N = int(1e8), 4
dd = model.generate(2026, V, N, np.full(3, 0.2), 100.0*np.eye(3), 100.0)
r0, mu0, D0 = dd.download(); dd.close()
r = _lib.pinned_empty((V,)); mu = _lib.pinned_empty((V,)); D = _lib.pinned_empty((V, 3))
r[:], mu[:], D[:] = r0, mu0, D0
hp = model.default_hyperparams(N)
for it in range(3):
    ds = model.Dataset(r=r, mu=mu, D=D, n_networks=N)
    t0 = time.perf_counter(); h = vb.device_dataset(ds); t1 = time.perf_counter()
    st, tr = vb.vb_fit(ds, hp); _ = st.k0k; t2 = time.perf_counter()
    print(f"upload {1e3*(t1-t0):.1f} ms, fit {1e3*(t2-t1):.1f} ms ({len(tr)} sweeps, {1e3*(t2-t1)/len(tr):.3f} ms/sweep)")
    del ds, st, tr, h
