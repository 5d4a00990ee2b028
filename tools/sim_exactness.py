import numpy as np, sys
sys.path.insert(0, '.')
from tests.golden_io import load
from tests.test_gpu_sim import _golden_state, _sim
g = load("sim"); ks = list(range(int(g["n_cases"])))
st = _golden_state(g, ks)
n = max(len(g[f"s{k}_ctrl"]) for k in ks)
ctrl = np.zeros((len(ks), n, 2))
for s, k in enumerate(ks):
    c = g[f"s{k}_ctrl"]; ctrl[s, :len(c)] = c; ctrl[s, len(c):] = c[-1]
done, snap = _sim().run(st, ctrl, n, snapshots=True)
for s, k in enumerate(ks):
    nt = len(g[f"s{k}_ctrl"]); nv = int(st.n_veh[s]); worst = 0; nexact = 0
    for t in range(nt):
        rec = snap[s, t]; ge = g[f"s{k}_ego"][t]; gv = g[f"s{k}_veh"][t]
        d = max(np.abs(rec[1:7] - ge[:6]).max(), np.abs(rec[8:8+4*nv].reshape(nv, 4) - gv[:, :4]).max())
        worst = max(worst, d); nexact += d == 0
    print(k, "max abs diff", worst, "bit-exact ticks", nexact, "/", nt)
