"""Sweeps to the reference stop rule on the 1695-sweep Table-1 golden for each storage mode."""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from golden_io import Golden
from paper_2401_10068_b200 import model, vb
g = Golden("fit_n3_v4000_t1")
r, mu, D = g.data()
ds = model.Dataset(r=r, mu=mu, D=D, n_networks=3)
h = g.hyper
hp = model.HyperParams(a0=h.a0, b0=h.b0, q0=h.q0, n0=h.n0, K0=h.K0, Lambda0=h.Lambda0)
for st_ in ("f64", "f32", "f32m"):
    st, tr = vb.vb_fit(vb.device_dataset(ds, storage=st_), hp, **g.fit_kw)
    print(st_, "sweeps", len(tr), "reference", int(g["n_iter"]), "max rel elbo err", float(np.max(np.abs(tr.elbo - g["elbo"][:len(tr)]) / np.abs(g["elbo"][:len(tr)]))))
