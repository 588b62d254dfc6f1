"""CPU restatement of the reference's training step -- TEST INFRASTRUCTURE
ONLY (the checker of the GPU training path; nothing under
paper_2305_16432_b200/ imports it).

Restates, in plain numpy fp64 with a hand-written reverse pass (no tape):
  * tuple_loss + ad.backward for the data loss (train.py:104-150, 189-205):
    forward of gnn.py:227-263, symmetrize (gnn.py:284-296),
    apply_learned_factor / loss_data, the x0-head auxiliary term, and the
    backward rules of autodiff.py:113-253 (affine, relu, mul, concat,
    gather_rows, segment_sum, flatten, sum_sq, sub, scale, add);
  * the minibatch mean in tuple-index order (train.py:208-226);
  * adam_step (train.py:164-185).
Pinned against gradients produced by pcgkit itself: tests/golden/train_*.npz
(tests/golden/make_golden_train.py), tests/test_train_oracle.py.
"""
import numpy as np

from . import port


def _relu(x):
    return np.where(x > 0.0, x, 0.0)


def forward_stash(hp, params, g):
    """gnn.forward (gnn.py:227-263, reference mode) keeping what the reverse
    pass needs. Returns (M, x0 or None, stash)."""
    node_in, edge_in = g.node_in, g.edge_in
    if hp.normalize:
        node_in = (node_in - g.node_stats[0]) / g.node_stats[1]
        edge_in = (edge_in - g.edge_stats[0]) / g.edge_stats[1]
    st = {"node_in": node_in, "edge_in": edge_in, "rounds": []}

    def mlp(prefix, x):  # l = l_mp = 1: one hidden layer
        h = _relu(port._affine(x, params[f"{prefix}.0.w"], params[f"{prefix}.0.b"]))
        return h, port._affine(h, params[f"{prefix}.1.w"], params[f"{prefix}.1.b"])

    st["h_ne"], v = mlp("node_enc", node_in)
    st["h_ee"], e = mlp("edge_enc", edge_in)
    for r in range(hp.n_mp):
        rd = {"v": v, "e": e}
        agg = port._segment_sum(e * v[g.dst], g.src, g.n)
        rd["agg"] = agg
        rd["hn"], v = mlp(f"mp{r}.node", np.concatenate((v, agg), axis=1))
        rd["v_new"] = v
        rd["he"], e = mlp(f"mp{r}.edge", np.concatenate((e, v[g.src], v[g.dst]), axis=1))
        st["rounds"].append(rd)
    st["e_out"], st["v_out"] = e, v
    st["h_ed"], M = mlp("edge_dec", e)
    x0 = None
    if hp.with_x0_head:
        st["h_nd"], x0 = mlp("node_dec", v)
        x0 = x0.reshape(-1)
    return M.reshape(-1), x0, st


def apply_factor(lv, rows, cols, diag, x):
    """(I+L') D (I+L')^T x, train.py:118-124: returns (w, y)."""
    u = x.copy()
    np.add.at(u, cols, lv * x[rows])
    w = diag * u
    y = w.copy()
    np.add.at(y, rows, lv * w[cols])
    return w, y


def tuple_loss_and_grad(hp, params, A, b, x, x0_aux_weight=0.1):
    """Loss (train.py:189-205, data loss) and d loss / d params for one
    tuple, as ad.backward would leave them in fwd.param_tensors[*].grad."""
    b = np.asarray(b, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    g = port.graph_from_system(A, b)
    M, x0, st = forward_stash(hp, params, g)
    low = np.flatnonzero(g.src > g.dst)  # lower edges in CSR order (gnn.py:284-296)
    lv = 0.5 * (M[low] + M[g.pair[low]])
    rows, cols = g.src[low], g.dst[low]
    diag = port.diagonal(A)
    w, y = apply_factor(lv, rows, cols, diag, x)
    res = y - b
    loss = float(res @ res)
    # ---- reverse pass
    gy = 2.0 * res  # sum_sq, sub
    t = gy.copy()
    np.add.at(t, cols, lv * gy[rows])
    dlv = gy[rows] * w[cols] + x[rows] * (diag * t)[cols]  # train.py:133-139
    dM = np.zeros_like(M)
    np.add.at(dM, low, 0.5 * dlv)
    np.add.at(dM, g.pair[low], 0.5 * dlv)
    grads = {}

    def mlp_back(prefix, x_in, h, dy):
        """Backward of a one-hidden-layer MLP; returns d x_in."""
        W1, W0 = params[f"{prefix}.1.w"], params[f"{prefix}.0.w"]
        grads[f"{prefix}.1.w"] = h.T @ dy
        grads[f"{prefix}.1.b"] = dy.sum(axis=0)
        dh = (dy @ W1.T) * (h > 0.0)
        grads[f"{prefix}.0.w"] = x_in.T @ dh
        grads[f"{prefix}.0.b"] = dh.sum(axis=0)
        return dh @ W0.T

    F = st["e_out"].shape[1]
    de = mlp_back("edge_dec", st["e_out"], st["h_ed"], dM[:, None])
    dv = np.zeros_like(st["v_out"])
    if hp.with_x0_head:
        aux = x0 - x
        loss = loss + x0_aux_weight * float(aux @ aux)
        dx0 = x0_aux_weight * (2.0 * aux)
        dv = dv + mlp_back("node_dec", st["v_out"], st["h_nd"], dx0[:, None])
    for r in range(hp.n_mp - 1, -1, -1):
        rd = st["rounds"][r]
        xe = np.concatenate((rd["e"], rd["v_new"][g.src], rd["v_new"][g.dst]), axis=1)
        dxe = mlp_back(f"mp{r}.edge", xe, rd["he"], de)
        de_prev = dxe[:, :F]
        dvn = dv.copy()
        np.add.at(dvn, g.src, dxe[:, F:2 * F])
        np.add.at(dvn, g.dst, dxe[:, 2 * F:])
        xn = np.concatenate((rd["v"], rd["agg"]), axis=1)
        dxn = mlp_back(f"mp{r}.node", xn, rd["hn"], dvn)
        dv_prev, dagg = dxn[:, :F], dxn[:, F:]
        dmsg = dagg[g.src]  # segment_sum backward
        de_prev = de_prev + dmsg * rd["v"][g.dst]
        dv_prev = dv_prev.copy()
        np.add.at(dv_prev, g.dst, dmsg * rd["e"])
        de, dv = de_prev, dv_prev
    mlp_back("edge_enc", st["edge_in"], st["h_ee"], de)
    mlp_back("node_enc", st["node_in"], st["h_ne"], dv)
    for name in params:  # parameters the loss does not reach (node_dec without the head term)
        grads.setdefault(name, None)
    return loss, grads


def batch_gradients(hp, params, tuples, indices, x0_aux_weight=0.1):
    """train.py:208-226: mean loss and mean gradients, tuple-index order."""
    total, sums = 0.0, {}
    for i in indices:
        A, b, x = tuples[i]
        loss, grads = tuple_loss_and_grad(hp, params, A, b, x, x0_aux_weight)
        total += loss
        for name, gr in grads.items():
            if gr is None:
                continue
            if name in sums:
                sums[name] += gr
            else:
                sums[name] = gr.copy()
    inv = 1.0 / len(indices)
    return total * inv, {k: v * inv for k, v in sums.items()}


def adam_step(params, grads, state, t, learning_rate=1e-3, beta1=0.9, beta2=0.999, eps=1e-8):
    """train.py:164-185 (state: dict with 'm' and 'v' dicts)."""
    bc1 = 1.0 - beta1 ** t
    bc2 = 1.0 - beta2 ** t
    for name in sorted(params):
        gr = grads.get(name)
        if gr is None:
            gr = np.zeros_like(params[name])
        if not np.all(np.isfinite(gr)):
            raise FloatingPointError(f"non-finite gradient for {name}")
        m = state["m"].get(name)
        if m is None:
            m = state["m"][name] = np.zeros_like(params[name])
            state["v"][name] = np.zeros_like(params[name])
        v = state["v"][name]
        m += (1.0 - beta1) * (gr - m)
        v += (1.0 - beta2) * (gr * gr - v)
        params[name] -= learning_rate * (m / bc1) / (np.sqrt(v / bc2) + eps)


def train(hp, params, tuples, batch_size=16, epochs=1, seed=0, learning_rate=1e-3, x0_aux_weight=0.1):
    """train.py:229-284 without the file outputs: returns (params, [batch losses])."""
    params = {k: v.copy() for k, v in params.items()}
    rng = np.random.default_rng(seed)
    state = {"m": {}, "v": {}}
    losses, step = [], 0
    for _ in range(epochs):
        order = rng.permutation(len(tuples))
        for lo in range(0, len(order), batch_size):
            batch = order[lo: lo + batch_size]
            loss, grads = batch_gradients(hp, params, tuples, batch, x0_aux_weight)
            step += 1
            adam_step(params, grads, state, step, learning_rate)
            losses.append(loss)
    return params, losses
