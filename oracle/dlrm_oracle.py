"""CPU restatement of the reference's TT-DLRM training step — TEST
INFRASTRUCTURE ONLY (tests/ and bench.py's CPU-baseline legs).

Follows /root/reference/pkg/src/ttemb/model.py:
  Mlp.forward / backward              model.py:153-172
  feature_interaction (+ backward)    model.py:107-131
  FieldTable.lookup / grads           model.py:208-243 (TT branch through
                                      ttb_oracle.forward / core_grads with the
                                      forward's reuse buffer borrowed, 238-239)
  DlrmModel.loss_and_grads            model.py:322-345
  DlrmModel.train_step                model.py:347-365 (fp64 velocity per
                                      parameter, one rounding into the param)
  loss_and_logit_grad (bce / mse)     model.py:71-86

Pinning: tests/test_oracle_golden.py runs three steps from the golden initial
parameters of tests/golden/dlrm.npz / dlrm_tc.npz (made by the unmodified
reference, tests/golden/make_golden.py) and compares losses and parameters.

Parameters are a dict name -> numpy array keyed like the reference's
named_params ("field_{f}.core{k}", "field_{f}.rows", "bottom.{i}.w", ...);
`fields` is a list of ttb_oracle.Geometry (TT field) or None (dense field).
"""
from __future__ import annotations

import numpy as np

from . import ttb_oracle as O


def sigmoid(z):
    """Stable logistic — model.py:68-75."""
    out = np.empty_like(z, dtype=np.float64)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def loss_and_logit_grad(z, y, kind="bce"):
    """model.py:78-86 (the loss clamps p, the gradient uses the raw sigmoid)."""
    if kind == "bce":
        p = np.clip(sigmoid(z), 1e-7, 1.0 - 1e-7)
        loss = float(-np.mean(y * np.log(p) + (1.0 - y) * np.log(1.0 - p)))
        return loss, (sigmoid(z) - y) / z.size
    return float(np.mean((z - y) ** 2)), 2.0 * (z - y) / z.size


def _mlp_names(params, prefix):
    n = 0
    while f"{prefix}.{n}.w" in params:
        n += 1
    return n


def mlp_forward(params, prefix, x):
    """model.py:153-161: ReLU between layers, linear output."""
    n = _mlp_names(params, prefix)
    inputs, pre = [], []
    for i in range(n):
        inputs.append(x)
        z = x @ params[f"{prefix}.{i}.w"] + params[f"{prefix}.{i}.b"]
        pre.append(z)
        x = np.maximum(z, 0.0) if i < n - 1 else z
    return x, (inputs, pre)


def mlp_backward(params, prefix, cache, gy, grads):
    """model.py:163-172; writes gw / gb into `grads`, returns d input."""
    inputs, pre = cache
    n = len(inputs)
    g = gy
    for i in range(n - 1, -1, -1):
        if i < n - 1:
            g = g * (pre[i] > 0)
        grads[f"{prefix}.{i}.w"] = inputs[i].T @ g
        grads[f"{prefix}.{i}.b"] = g.sum(axis=0)
        g = g @ params[f"{prefix}.{i}.w"].T
    return g


def interaction(vectors):
    """concat(v0, pairwise dots in lexicographic order) — model.py:107-114."""
    stack = np.stack(vectors, axis=1)
    gram = stack @ stack.transpose(0, 2, 1)
    iu = np.triu_indices(stack.shape[1], k=1)
    return np.concatenate([vectors[0], gram[:, iu[0], iu[1]]], axis=1)


def interaction_backward(vectors, gout):
    """model.py:117-131."""
    stack = np.stack(vectors, axis=1)
    v, d = stack.shape[1], vectors[0].shape[1]
    iu = np.triu_indices(v, k=1)
    gp = np.zeros((stack.shape[0], v, v), dtype=gout.dtype)
    gp[:, iu[0], iu[1]] = gout[:, d:]
    gstack = (gp + gp.transpose(0, 2, 1)) @ stack
    grads = [gstack[:, i].copy() for i in range(v)]
    grads[0] += gout[:, :d]
    return grads


def loss_and_grads(params, fields, dense, sparse, labels, loss="bce"):
    """model.py:272-345 for one batch: sparse[f] = (idx (T,), offsets (B+1,))."""
    dtype = params["bottom.0.w"].dtype
    x = dense.astype(dtype, copy=False)
    v0, bcache = mlp_forward(params, "bottom", x)
    vectors, ctx = [v0], []
    for f, geom in enumerate(fields):
        idx, off = sparse[f]
        if geom is not None:  # TT field: reuse plan + buffer (model.py:210-219)
            cores = [params[f"field_{f}.core{k}"] for k in range(geom.d)]
            out, plan = O.forward(cores, geom, idx, off, want_plan=True)
            ctx.append(plan)
        else:  # dense field (model.py:220-229)
            rows = params[f"field_{f}.rows"]
            if idx.size and (idx.min() < 0 or idx.max() >= rows.shape[0]):
                raise ValueError(f"index outside [0, {rows.shape[0]})")
            bag = np.repeat(np.arange(off.size - 1), np.diff(off))
            out = np.zeros((off.size - 1, rows.shape[1]), dtype=rows.dtype)
            np.add.at(out, bag, rows[idx])
            ctx.append(None)
        vectors.append(out)
    z, tcache = mlp_forward(params, "top", interaction(vectors))
    z = z.reshape(-1)
    lval, gz = loss_and_logit_grad(z, labels, loss)
    grads = {}
    gi = mlp_backward(params, "top", tcache, gz.reshape(-1, 1).astype(dtype), grads)
    gv = interaction_backward(vectors, gi)
    mlp_backward(params, "bottom", bcache, gv[0], grads)
    for f, geom in enumerate(fields):
        idx, off = sparse[f]
        per_occ = np.repeat(gv[f + 1], np.diff(off), axis=0)
        if geom is not None:  # model.py:234-240
            cores = [params[f"field_{f}.core{k}"] for k in range(geom.d)]
            rows, ug = O.unique_aggregate(idx, per_occ)
            plan = ctx[f]
            borrowed = (plan["work"], plan["slots"]) if geom.d == 3 else None
            for k, gk in enumerate(O.core_grads(cores, geom, rows, ug, borrowed=borrowed)):
                grads[f"field_{f}.core{k}"] = gk
        else:  # model.py:241-243
            rows = params[f"field_{f}.rows"]
            g = np.zeros(rows.shape, dtype=np.float64)
            np.add.at(g, idx, per_occ.astype(np.float64))
            grads[f"field_{f}.rows"] = g
    return lval, grads


def train_step(params, fields, dense, sparse, labels, lr, momentum, velocity, loss="bce"):
    """model.py:347-365: SGD(+momentum) on every parameter, fp64 velocity,
    one rounding into the parameter dtype. Updates params / velocity in place."""
    lval, grads = loss_and_grads(params, fields, dense, sparse, labels, loss)
    for name, p in params.items():
        g = np.asarray(grads[name], dtype=np.float64)
        if momentum > 0.0:
            v = velocity.get(name)
            if v is None:
                v = velocity[name] = np.zeros(p.shape, dtype=np.float64)
            v *= momentum
            v += g
            g = v
        np.subtract(p, lr * g, out=p, casting="same_kind")
    return lval


def init_params(rows_per_field, emb_dim, ranks, tt_threshold, n_dense, bottom, top, seed=0, dtype=np.float32):
    """Shapes of the reference's DlrmModel (model.py:248-268) with seeded
    random values — for CPU timing samples only (the golden tests start from
    the reference's own initial parameters)."""
    rng = np.random.default_rng(seed)
    params, fields = {}, []
    d = len(ranks) - 1
    for f, rows in enumerate(rows_per_field):
        if rows >= tt_threshold:
            m, n = O.factorize(rows, emb_dim, d)
            g = O.Geometry(tuple(m), tuple(n), tuple(ranks))
            for k, c in enumerate(O.init_cores(g, int(rng.integers(2 ** 31)), dtype=dtype)):
                params[f"field_{f}.core{k}"] = c
            fields.append(g)
        else:
            params[f"field_{f}.rows"] = (rng.standard_normal((rows, emb_dim)) * 0.1).astype(dtype)
            fields.append(None)
    v = len(rows_per_field) + 1
    inter = emb_dim + v * (v - 1) // 2
    for prefix, sizes in (("bottom", (n_dense, *bottom, emb_dim)), ("top", (inter, *top, 1))):
        for i, (a, b) in enumerate(zip(sizes[:-1], sizes[1:])):
            params[f"{prefix}.{i}.w"] = (rng.standard_normal((a, b)) * np.sqrt(2.0 / a)).astype(dtype)
            params[f"{prefix}.{i}.b"] = np.zeros(b, dtype=dtype)
    return params, fields
