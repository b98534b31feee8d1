"""Pins of the CPU oracle against what the paper and the mathematics fix
(pins P1-P8).  None of these compare the oracle with itself:
each uses a closed form, an independent formulation (textbook Eq. 1/4/5, torch
autograd of an independently written loss, a literal Eq. 7 shift), finite
differences of the oracle's own loss value, or an invariant."""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from oracle import BF16, F32, Pool

GOLD = os.path.join(os.path.dirname(__file__), "golden", "closed_forms.json")


def _pool_from(rows, dtype=F32):
    d = len(rows[0][0])
    p = Pool(len(rows), d, dtype)
    for vec, lab in rows:  # one enqueue per slot, oldest first
        G = np.array([vec], dtype=np.float32) if dtype == F32 else oracle.f64_to_bf16(np.array([vec]))
        p.enqueue(G, np.array([lab]))
    return p


# ----------------------------------------------------------------------------- P4/P5
@pytest.mark.parametrize("case", json.load(open(GOLD))["cases"], ids=lambda c: c["id"])
def test_closed_forms(case):
    p = _pool_from(case["pool"])
    X = np.array(case["x"], dtype=np.float32)
    r = p.loss(X, np.array(case["y"]), None, case["s"], case["m"])
    # inputs are stored as fp32 (0.6, 0.8 are not exact), and s=64 amplifies that
    # rounding (|dz| <= 64 * 2^-24 per unit input): tolerances reflect it.
    assert r.L == pytest.approx(case["L"], rel=5e-6, abs=1e-9)
    if case["dx"] is not None:
        np.testing.assert_allclose(r.dx, np.array(case["dx"]), rtol=5e-6, atol=1e-9)


@pytest.mark.parametrize("case", json.load(open(GOLD))["dT_cases"], ids=lambda c: c["id"])
def test_closed_form_pool_gradient(case):
    p = _pool_from(case["pool"])
    r = p.loss(np.array(case["x"], np.float32), np.array(case["y"]), None, case["s"], case["m"],
               want_dT=True)
    np.testing.assert_allclose(r.dT, np.array(case["dT"]), atol=1e-12)


def test_duplicate_target_is_newest_and_slot_order_irrelevant():
    """D8: with the slot contents permuted but the write order (seq) kept, the
    loss is unchanged (case F enqueued in a different physical order)."""
    rows = json.load(open(GOLD))["cases"][4]["pool"]
    base = _pool_from(rows).loss(np.array([[1.0, 0.0]], np.float32), np.array([7]), None, 64, 0.35)
    # wrap the ring so the same four rows (same write order) land in rotated slots
    p = Pool(4, 2, F32)
    p.enqueue(np.zeros((2, 2), np.float32), np.array([100, 101]))  # will be overwritten
    for vec, lab in rows:
        p.enqueue(np.array([vec], np.float32), np.array([lab]))
    r = p.loss(np.array([[1.0, 0.0]], np.float32), np.array([7]), None, 64, 0.35)
    assert r.L == pytest.approx(base.L, rel=1e-14)
    assert r.tslot[0] == 0  # newest label-7 row was written 5th -> slot (2+2) % 4 = 0
    np.testing.assert_allclose(r.dx, base.dx, rtol=1e-13)


# ----------------------------------------------------------------------------- P1
def _logsumexp(a, axis=-1):
    mx = np.max(a, axis=axis, keepdims=True)
    return (mx + np.log(np.sum(np.exp(a - mx), axis=axis, keepdims=True))).squeeze(axis)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_eq4_reduces_to_eq1_full_softmax(seed):
    """P1: pool = the full classifier W (all n_ID classes, distinct labels), s=1,
    m=0 -> L equals the textbook full-softmax CE of Eq. 1 on x_hat."""
    rng = np.random.default_rng(seed)
    n_id, d, N = 37, 6, 9
    W = rng.standard_normal((n_id, d)).astype(np.float32)
    X = rng.standard_normal((N, d)).astype(np.float32)
    y = rng.integers(0, n_id, N)
    p = Pool(n_id, d, F32)
    p.enqueue(W, np.arange(n_id))
    r = p.loss(X, y, None, 1.0, 0.0)
    Xh = X.astype(np.float64) / np.linalg.norm(X.astype(np.float64), axis=1, keepdims=True)
    logits = Xh @ W.astype(np.float64).T                       # W_j^T x_i
    L_eq1 = -np.mean(logits[np.arange(N), y] - _logsumexp(logits))
    assert r.N_pos == N and r.N_neg == 0
    assert abs(r.L - L_eq1) <= 1e-12


# ----------------------------------------------------------------------------- P2
def test_masked_softmax_eq4_eq5_and_autograd_dx():
    """P2: pool = {W_j : nu_j = 1} with every batch label selected (Eq. 3).
    Oracle L == Eq. 4; oracle dL/dT_k == Eq. 5 for the selected
    classifiers; oracle dx == torch autograd of Eq. 4 through x_hat = x/||x||."""
    rng = np.random.default_rng(5)
    n_id, d, N, C = 50, 7, 8, 20
    W = rng.standard_normal((n_id, d)).astype(np.float32)
    X = rng.standard_normal((N, d)).astype(np.float32)
    y = rng.choice(n_id, N, replace=True)
    sel = set(y.tolist())
    rest = [j for j in range(n_id) if j not in sel]
    sel = sorted(sel | set(rng.choice(rest, C - len(sel), replace=False).tolist()))
    nu = np.zeros(n_id)
    nu[sel] = 1.0
    p = Pool(C, d, F32)
    p.enqueue(W[sel], np.array(sel))
    r = p.loss(X, y, None, 1.0, 0.0, want_dT=True)

    X64, W64 = X.astype(np.float64), W.astype(np.float64)
    Xh = X64 / np.linalg.norm(X64, axis=1, keepdims=True)
    logits = Xh @ W64.T
    masked = np.where(nu[None, :] > 0, logits, -np.inf)
    L_eq4 = -np.mean(logits[np.arange(N), y] - _logsumexp(masked))
    assert abs(r.L - L_eq4) <= 1e-12 * max(1.0, abs(L_eq4))

    # Eq. 5: dL/dW_k = -1/N sum_i (delta_{k y_i} - nu_k p_ik) x_i
    phat = np.exp(masked - _logsumexp(masked)[:, None])
    dW = np.zeros_like(W64)
    for k in range(n_id):
        for i in range(N):
            dW[k] += -(1.0 / N) * ((1.0 if y[i] == k else 0.0) - nu[k] * phat[i, k]) * Xh[i]
    np.testing.assert_allclose(r.dT, dW[sel], rtol=1e-8, atol=1e-13)

    xt = torch.tensor(X64, requires_grad=True)
    xh = xt / xt.norm(dim=1, keepdim=True)
    lg = xh @ torch.tensor(W64).T
    lg = lg.masked_fill(torch.tensor(nu)[None, :] == 0, -float("inf"))
    loss = torch.nn.functional.cross_entropy(lg, torch.tensor(y))
    loss.backward()
    np.testing.assert_allclose(r.dx, xt.grad.numpy(), rtol=1e-8, atol=1e-13)


def test_margin_scale_dups_outofpool_vs_autograd():
    """P2': full definition with s, m, duplicate labels and out-of-pool rows; the
    oracle's hand-derived gradient equals torch autograd of an independently
    written loss (targets = newest duplicate, D8)."""
    rng = np.random.default_rng(11)
    C, d = 12, 6
    T = rng.standard_normal((C, d)).astype(np.float32)
    lab = rng.integers(0, 5, C)
    p = Pool(C, d, F32)
    p.enqueue(T, lab)
    N = 7
    X = (rng.standard_normal((N, d)) * 2).astype(np.float32)
    y = np.array([0, 1, 2, 3, 4, 9, 11])
    s, m = 30.0, 0.2
    r = p.loss(X, y, None, s, m)
    # independent formulation
    tgt = []
    for i in range(N):
        hits = [c for c in range(C) if lab[c] == y[i]]
        tgt.append(max(hits) if hits else -1)  # single fill: seq == slot, newest = largest
    np.testing.assert_array_equal(r.tslot, tgt)
    xt = torch.tensor(X.astype(np.float64), requires_grad=True)
    Tt = torch.tensor(T.astype(np.float64))
    cos = (xt / xt.norm(dim=1, keepdim=True)) @ Tt.T
    pos = [i for i in range(N) if tgt[i] >= 0]
    neg = [i for i in range(N) if tgt[i] < 0]
    z = s * cos
    ce = 0
    for i in pos:
        zi = z[i].clone()
        zi[tgt[i]] = zi[tgt[i]] - s * m
        ce = ce + torch.logsumexp(zi, 0) - zi[tgt[i]]
    loss = ce / len(pos) + sum(cos[i].mean() for i in neg) / len(neg)
    loss.backward()
    assert r.L == pytest.approx(loss.item(), rel=1e-12)
    np.testing.assert_allclose(r.dx, xt.grad.numpy(), rtol=1e-9, atol=1e-12)


# ----------------------------------------------------------------------------- P3
def test_finite_differences_of_oracle_loss():
    """P3: Richardson-extrapolated central differences of the oracle's L with
    respect to the raw x.  Inputs are dyadic so x +- h is exact in fp32."""
    rng = np.random.default_rng(3)
    C, d, N = 14, 8, 6
    T = (rng.integers(-128, 128, (C, d)) / 128.0).astype(np.float32)
    lab = rng.integers(0, 6, C)
    p = Pool(C, d, F32)
    p.enqueue(T, lab)
    X = (rng.integers(-256, 256, (N, d)) / 128.0).astype(np.float32)
    X[0] *= 3  # ||x|| != 1
    y = np.array([0, 1, 2, 3, 7, 8])  # some in-pool (incl. duplicates), some out-of-pool
    s, m = 16.0, 0.35
    r = p.loss(X, y, None, s, m)
    assert r.N_pos >= 2 and r.N_neg >= 1

    def L(Xp):
        return p.loss(Xp, y, None, s, m).L

    h = 2.0 ** -8
    num = np.zeros_like(r.dx)
    for i in range(N):
        for k in range(d):
            def D(hh):
                Xa, Xb = X.copy(), X.copy()
                Xa[i, k] += hh
                Xb[i, k] -= hh
                return (L(Xa) - L(Xb)) / (2 * hh)
            num[i, k] = (4 * D(h / 2) - D(h)) / 3
    np.testing.assert_allclose(r.dx, num, rtol=1e-6, atol=1e-8)


# ----------------------------------------------------------------------------- P6
def test_invariants_softmax_rows_cosines_and_permutation():
    """P6: sum_c p_ic = 1; cos in [-1,1] on fp64-unit data (phi in [-1,1], ell >= 0);
    row-permutation equivariance."""
    rng = np.random.default_rng(9)
    C, d, N = 40, 16, 10
    T = rng.standard_normal((C, d))
    T /= np.linalg.norm(T, axis=1, keepdims=True)
    p = Pool(C, d, F32)
    p.enqueue(T.astype(np.float32), rng.integers(0, 8, C))
    X = rng.standard_normal((N, d)).astype(np.float32)
    y = np.concatenate([rng.integers(0, 8, 6), np.arange(100, 104)])
    r = p.loss(X, y, None, 64.0, 0.35, want_P=True)
    pos = r.tslot >= 0
    np.testing.assert_allclose(r.P[pos].sum(axis=1), 1.0, atol=1e-12)
    assert np.all(r.ell[pos] >= 0)
    assert np.all(np.abs(r.phi) <= 1.0 + 1e-6)
    perm = rng.permutation(N)
    r2 = p.loss(X[perm], y[perm], None, 64.0, 0.35)
    assert r2.L == pytest.approx(r.L, rel=1e-13)
    np.testing.assert_allclose(r2.dx, r.dx[perm], rtol=1e-12, atol=1e-15)


def test_loss_rows_matches_full():
    rng = np.random.default_rng(4)
    C, d, N = 30, 8, 12
    p = Pool(C, d, BF16)
    p.enqueue(oracle.f64_to_bf16(rng.standard_normal((C, d))), rng.integers(0, 6, C))
    X = oracle.f64_to_bf16(rng.standard_normal((N, d)))
    y = rng.integers(0, 9, N)
    full = p.loss(X, y, None, 64.0, 0.35)
    rows = np.array([11, 0, 5])
    sub = p.loss_rows(X, y, None, 64.0, 0.35, rows)
    np.testing.assert_allclose(sub["dx"], full.dx[rows], rtol=1e-14)
    np.testing.assert_allclose(sub["lse"], full.lse[rows], rtol=1e-14)
    assert sub["N_pos"] == full.N_pos


def test_pairing_check_and_errors():
    p = Pool(8, 2, F32)
    p.enqueue(np.eye(2, dtype=np.float32).repeat(2, 0), np.array([1, 2, 3, 4]))
    X = np.array([[1, 0], [0, 1]], np.float32)
    p.loss(X, np.array([3, 9]), np.array([2, -1], np.int32), 64, 0.35)  # row 0 paired to block row 2
    with pytest.raises(oracle.OracleError) as e:
        p.loss(X, np.array([3, 9]), np.array([1, -1], np.int32), 64, 0.35)
    assert e.value.code == 4
    with pytest.raises(oracle.OracleError):
        p.loss(np.zeros((1, 2), np.float32), np.array([1]), None, 64, 0.35)  # zero row
    with pytest.raises(oracle.OracleError) as e:
        p.enqueue(np.zeros((9, 2), np.float32), np.arange(9))
    assert e.value.code == 3


# ----------------------------------------------------------------------------- P7
def _literal_shift(T, lab, occ, G, y):
    """Eq. 7 literally plus Algorithm 1's fill branch:
    an array of C rows; the first `occ` are occupied, oldest first."""
    C, M = len(lab), len(y)
    if occ + M <= C:            # fill unoccupied positions sequentially
        T[occ:occ + M] = G
        lab[occ:occ + M] = y
        return occ + M
    # shift out the oldest rows, append the new block at the end
    k = occ + M - C
    T[:occ - k] = T[k:occ].copy()
    lab[:occ - k] = lab[k:occ].copy()
    T[C - M:] = G
    lab[C - M:] = y
    return C


def test_enqueue_spec_example_and_wrap():
    """A,B / C,D / E,F at C=4 -> slots [E,F,C,D]; wrap at C=5, M=2 -> [F,B,C,D,E]
    which as a ring read from the oldest equals the literal shift [B,C,D,E,F]."""
    p = Pool(4, 1, F32)
    for blk in ([1, 2], [3, 4], [5, 6]):
        p.enqueue(np.array(blk, np.float32)[:, None], np.array(blk))
    assert p.lab.tolist() == [5, 6, 3, 4]
    p = Pool(5, 1, F32)
    for blk in ([1, 2], [3, 4], [5, 6]):
        p.enqueue(np.array(blk, np.float32)[:, None], np.array(blk))
    assert p.lab.tolist() == [6, 2, 3, 4, 5]
    head = int(p.E[0]) % 5
    assert np.roll(p.lab, -head).tolist() == [2, 3, 4, 5, 6]


def test_enqueue_equals_literal_shift_random():
    """10^3 random blocks of random M <= C at C <= 64; the ring read
    from its oldest slot equals a literal Eq. 7 shift implementation."""
    rng = np.random.default_rng(1)
    for trial in range(4):
        C, d = int(rng.integers(1, 65)), 3
        p = Pool(C, d, F32)
        T_lit = np.zeros((C, d), np.float32)
        lab_lit = np.full(C, -1, np.int64)
        occ = 0
        for it in range(250):
            M = int(rng.integers(1, C + 1))
            G = rng.standard_normal((M, d)).astype(np.float32)
            y = rng.integers(0, 10**6, M)
            p.enqueue(G, y)
            occ = _literal_shift(T_lit, lab_lit, occ, G, y)
            E = int(p.E[0])
            if E < C:
                order = np.arange(E)
            else:
                order = (np.arange(C) + E) % C  # oldest first
            np.testing.assert_array_equal(p.T[order], T_lit[:occ])
            np.testing.assert_array_equal(p.lab[order], lab_lit[:occ])


def test_residency_and_last_blocks():
    """P:207 / S:279 / S:311: with M | C every row stays exactly C/M enqueues; after
    k enqueues the pool holds exactly the last ceil(C/M) blocks in order (BJ:5)."""
    C, M = 12, 3
    p = Pool(C, 1, F32)
    first_seen, last_seen = {}, {}
    for k in range(1, 20):
        ids = np.arange((k - 1) * M, k * M)
        p.enqueue(ids.astype(np.float32)[:, None], ids)
        for v in p.lab[: min(k * M, C)]:
            first_seen.setdefault(int(v), k)
            last_seen[int(v)] = k
        nb = math.ceil(C / M)
        want = np.arange(max(0, k - nb) * M, k * M)
        assert sorted(p.lab[: min(k * M, C)].tolist()) == want.tolist()
    for v in range(0, 10 * M):
        assert last_seen[v] - first_seen[v] + 1 == C // M


# ----------------------------------------------------------------------------- P8
def test_ema_boundaries_and_closed_form():
    """S:220-222 boundaries, S:510 closed form after n steps, S:227 contraction."""
    rng = np.random.default_rng(0)
    th = rng.standard_normal(1000).astype(np.float32)
    ph = rng.standard_normal(1000).astype(np.float32)
    np.testing.assert_array_equal(oracle.ema(th, ph, 0.0), th)
    np.testing.assert_array_equal(oracle.ema(th, ph, 1.0), ph)
    assert oracle.ema(np.zeros(1, np.float32), np.ones(1, np.float32), 0.999)[0] == np.float32(0.999)
    m = 0.9
    g = ph.copy()
    thetas = [rng.standard_normal(1000).astype(np.float32) for _ in range(25)]
    for t in thetas:
        g = oracle.ema(t, g, m)
    n = len(thetas)
    cf = m ** n * ph.astype(np.float64) + (1 - m) * sum(
        m ** i * thetas[n - 1 - i].astype(np.float64) for i in range(n))
    np.testing.assert_allclose(g, cf, rtol=0, atol=n * 2e-7 * np.abs(cf).max())
    g1 = oracle.ema(th, ph, 0.7)
    np.testing.assert_allclose(np.abs(g1.astype(np.float64) - th),
                               0.7 * np.abs(ph.astype(np.float64) - th), rtol=1e-6, atol=1e-6)


# ----------------------------------------------------------------------------- K = 2 (NEXT-1)
def _pool_k(slots, K=2):
    """slots: list of (K feature vectors, label), oldest first."""
    d = len(slots[0][0][0])
    p = Pool(len(slots), d, F32, K=K)
    for feats, lab in slots:
        p.enqueue(np.array([feats], np.float32), np.array([lab]))
    return p


def test_k2_spec_example_closed_form():
    """K=2 features with cosines 0.8 and 0.6 to the probe give the logit 0.7 (s=1).
    With a second slot orthogonal to x the CE is ln(1+e^-0.7) (Eq. 8 average + Eq. 9)."""
    p = _pool_k([([[0.8, 0.6, 0.0], [0.6, 0.0, 0.8]], 0), ([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0]], 1)])
    r = p.loss(np.array([[1.0, 0.0, 0.0]], np.float32), np.array([0]), None, 1.0, 0.0)
    assert r.L == pytest.approx(math.log1p(math.exp(-0.7)), rel=1e-6)


def test_k2_true_cosine_for_lcos():
    """R4: for K >= 2 L_cos uses cos(x, T_bar) = <x, T_bar>/||T_bar||;
    T_bar_0 = (0.7, 0.3, 0.4), T_bar_1 = (0, .5, .5) -> phi = 0.7/||T_bar_0|| / 2."""
    p = _pool_k([([[0.8, 0.6, 0.0], [0.6, 0.0, 0.8]], 0), ([[0.0, 1.0, 0.0], [0.0, 0.0, 1.0]], 1)])
    r = p.loss(np.array([[1.0, 0.0, 0.0]], np.float32), np.array([9]), None, 64.0, 0.35)
    assert r.L == pytest.approx(0.7 / math.sqrt(0.49 + 0.09 + 0.16) / 2.0, rel=1e-6)


def test_k2_cancelling_features_and_zero_center():
    """T[c,0] = -T[c,1] gives T_bar_c = 0: logit 0 for every row (uniform softmax
    with the margined target), and the zero-norm center contributes 0 to L_cos."""
    p = _pool_k([([[1.0, 0.0], [-1.0, 0.0]], 3), ([[0.0, 1.0], [0.0, -1.0]], 4)])
    r = p.loss(np.array([[0.6, 0.8]], np.float32), np.array([3]), None, 10.0, 0.0)
    assert r.L == pytest.approx(math.log(2.0), rel=1e-12)
    r = p.loss(np.array([[0.6, 0.8]], np.float32), np.array([7]), None, 10.0, 0.0)
    assert r.L == 0.0 and np.all(r.dx == 0.0)


def test_k2_duplicated_features_equal_k1():
    """Paper-literal insertion (one G-Net feature duplicated over K) reduces the
    K=2 pool to the K=1 pool (unit rows: true cosine == stored inner product)."""
    rng = np.random.default_rng(21)
    C, d = 20, 8
    T = rng.standard_normal((C, d))
    T /= np.linalg.norm(T, axis=1, keepdims=True)
    T = T.astype(np.float32)
    lab = rng.integers(0, 6, C)
    p1 = Pool(C, d, F32)
    p1.enqueue(T, lab)
    p2 = Pool(C, d, F32, K=2)
    p2.enqueue(np.stack([T, T], axis=1), lab)
    X = rng.standard_normal((9, d)).astype(np.float32)
    y = np.concatenate([rng.integers(0, 6, 6), [50, 51, 52]])
    a, b = p1.loss(X, y, None, 30.0, 0.2), p2.loss(X, y, None, 30.0, 0.2)
    assert b.L == pytest.approx(a.L, rel=1e-6)
    np.testing.assert_allclose(b.dx, a.dx, rtol=1e-5, atol=1e-8)


def test_k2_autograd_and_finite_differences():
    """K=2 gradient: oracle dx == torch autograd of an independent formulation (T_bar mean,
    margined CE on the newest duplicate, true-cosine L_cos) and == Richardson differences."""
    rng = np.random.default_rng(23)
    C, d, K = 11, 6, 2
    T = (rng.integers(-128, 128, (C, K, d)) / 128.0).astype(np.float32)
    lab = rng.integers(0, 5, C)
    p = Pool(C, d, F32, K=K)
    p.enqueue(T, lab)
    X = (rng.integers(-256, 256, (6, d)) / 128.0).astype(np.float32)
    y = np.array([0, 1, 2, 3, 8, 9])
    s, m = 16.0, 0.3
    r = p.loss(X, y, None, s, m)
    Tb = torch.tensor(T.astype(np.float64)).mean(dim=1)
    xt = torch.tensor(X.astype(np.float64), requires_grad=True)
    cos = (xt / xt.norm(dim=1, keepdim=True)) @ Tb.T
    tgt = [max([c for c in range(C) if lab[c] == y[i]], default=-1) for i in range(len(y))]
    pos = [i for i in range(len(y)) if tgt[i] >= 0]
    neg = [i for i in range(len(y)) if tgt[i] < 0]
    ce = 0
    for i in pos:
        zi = s * cos[i].clone()
        zi[tgt[i]] = zi[tgt[i]] - s * m
        ce = ce + torch.logsumexp(zi, 0) - zi[tgt[i]]
    tcos = cos / Tb.norm(dim=1)[None, :]
    loss = ce / len(pos) + sum(tcos[i].mean() for i in neg) / len(neg)
    loss.backward()
    assert r.L == pytest.approx(loss.item(), rel=1e-12)
    np.testing.assert_allclose(r.dx, xt.grad.numpy(), rtol=1e-9, atol=1e-12)
    h = 2.0 ** -8
    num = np.zeros_like(r.dx)
    for i in range(len(y)):
        for k in range(d):
            def D(hh):
                Xa, Xb = X.copy(), X.copy()
                Xa[i, k] += hh
                Xb[i, k] -= hh
                return (p.loss(Xa, y, None, s, m).L - p.loss(Xb, y, None, s, m).L) / (2 * hh)
            num[i, k] = (4 * D(h / 2) - D(h)) / 3
    np.testing.assert_allclose(r.dx, num, rtol=1e-6, atol=1e-8)


# ----------------------------------------------------------------------------- NEXT-3 phi variants
from oracle import PHI_MAX, PHI_MEAN, PHI_SUM  # noqa: E402


def test_phi_variants_spec_example():
    """C=2, F = T_bar_0 (unit), T_bar_1 orthogonal -> mean L_cos = 0.5; the sum is
    1.0 and the hardest negative (max) is 1.0.  With T_bar_1 = -F: mean 0, hinged mean 0.5,
    max 1, sum 0 (closed forms of the NEXT-3 reductions)."""
    F = [0.6, 0.8, 0.0]
    for other, want in (([0.0, 0.0, 1.0], {(PHI_MEAN, 0): 0.5, (PHI_SUM, 0): 1.0, (PHI_MAX, 0): 1.0,
                                             (PHI_MEAN, 1): 0.5, (PHI_MAX, 1): 1.0}),
                        ([-0.6, -0.8, 0.0], {(PHI_MEAN, 0): 0.0, (PHI_SUM, 0): 0.0, (PHI_MAX, 0): 1.0,
                                               (PHI_MEAN, 1): 0.5, (PHI_SUM, 1): 1.0})):
        p = _pool_from([(F, 0), (other, 1)])
        for (mode, hinge), L in want.items():
            r = p.loss(np.array([F], np.float32), np.array([5]), None, 64.0, 0.35, phi_mode=mode,
                       hinge=bool(hinge))
            assert r.L == pytest.approx(L, abs=1e-7), (other, mode, hinge)


def test_phi_max_hinge_all_negative_is_zero():
    """Hardest negative with the hinge: every cosine <= 0 -> phi = 0 and zero gradient."""
    p = _pool_from([([-1.0, 0.0], 0), ([0.0, -1.0], 1)])
    r = p.loss(np.array([[0.6, 0.8]], np.float32), np.array([9]), None, 64.0, 0.0, phi_mode=PHI_MAX,
               hinge=True)
    assert r.L == 0.0 and np.all(r.dx == 0.0)
    r = p.loss(np.array([[0.6, 0.8]], np.float32), np.array([9]), None, 64.0, 0.0, phi_mode=PHI_MAX)
    assert r.L == pytest.approx(-0.6, abs=1e-7)


def test_lambda_zero_is_ce_only():
    """lambda = 0 gives L_total = L_ce and zero gradient on out-of-pool rows;
    lambda scales L_cos and its gradient linearly."""
    rng = np.random.default_rng(31)
    C, d = 16, 8
    T = rng.standard_normal((C, d)); T /= np.linalg.norm(T, axis=1, keepdims=True)
    p = Pool(C, d, F32)
    p.enqueue(T.astype(np.float32), rng.integers(0, 5, C))
    X = rng.standard_normal((6, d)).astype(np.float32)
    y = np.array([0, 1, 2, 40, 41, 42])
    r1 = p.loss(X, y, None, 20.0, 0.3)
    r0 = p.loss(X, y, None, 20.0, 0.3, lam=0.0)
    r3 = p.loss(X, y, None, 20.0, 0.3, lam=3.0)
    neg = r1.tslot < 0
    assert r0.L == pytest.approx(r1.L_ce, rel=1e-14)
    assert np.all(r0.dx[neg] == 0.0)
    assert r3.L == pytest.approx(r1.L_ce + 3.0 * r1.L_cos, rel=1e-13)
    np.testing.assert_allclose(r3.dx[neg], 3.0 * r1.dx[neg], rtol=1e-13)
    np.testing.assert_array_equal(r3.dx[~neg], r1.dx[~neg])


@pytest.mark.parametrize("mode,hinge", [(PHI_SUM, False), (PHI_MAX, False), (PHI_MEAN, True),
                                        (PHI_SUM, True), (PHI_MAX, True)])
@pytest.mark.parametrize("K", [1, 2])
def test_phi_variants_autograd_and_finite_differences(mode, hinge, K):
    """Each variant's oracle gradient == torch autograd of an independent formulation
    (torch.max / relu over the true cosines) and == Richardson differences of the oracle's
    own loss value (inputs away from ties and from cos = 0)."""
    rng = np.random.default_rng(40 + mode * 2 + int(hinge) + 10 * K)
    C, d = 9, 5
    T = (rng.integers(-128, 128, (C, K, d)) / 128.0).astype(np.float32)
    lab = rng.integers(0, 4, C)
    p = Pool(C, d, F32, K=K)
    p.enqueue(T if K > 1 else T[:, 0], lab)
    X = (rng.integers(-256, 256, (6, d)) / 128.0).astype(np.float32)
    y = np.array([0, 1, 2, 7, 8, 9])
    s, m, lam = 12.0, 0.25, 0.7
    kw = dict(phi_mode=mode, hinge=hinge, lam=lam)
    r = p.loss(X, y, None, s, m, **kw)
    Tb = torch.tensor(T.astype(np.float64)).mean(dim=1)
    xt = torch.tensor(X.astype(np.float64), requires_grad=True)
    cos = (xt / xt.norm(dim=1, keepdim=True)) @ Tb.T
    tgt = [max([c for c in range(C) if lab[c] == y[i]], default=-1) for i in range(len(y))]
    pos = [i for i in range(len(y)) if tgt[i] >= 0]
    neg = [i for i in range(len(y)) if tgt[i] < 0]
    ce = 0
    for i in pos:
        zi = s * cos[i].clone()
        zi[tgt[i]] = zi[tgt[i]] - s * m
        ce = ce + torch.logsumexp(zi, 0) - zi[tgt[i]]
    # K = 1 keeps the stored rows as they are (D2); K >= 2 divides by ||T_bar|| (R4)
    tcos = cos / Tb.norm(dim=1)[None, :] if K > 1 else cos
    hc = torch.relu(tcos) if hinge else tcos
    red = {PHI_SUM: lambda v: v.sum(), PHI_MAX: lambda v: v.max()}[mode] if mode != PHI_MEAN else (lambda v: v.mean())
    loss = ce / len(pos) + lam * sum(red(hc[i]) for i in neg) / len(neg)
    loss.backward()
    assert r.L == pytest.approx(loss.item(), rel=1e-12)
    np.testing.assert_allclose(r.dx, xt.grad.numpy(), rtol=1e-9, atol=1e-12)
    h = 2.0 ** -10
    num = np.zeros_like(r.dx)
    for i in range(len(y)):
        for k in range(d):
            def D(hh):
                Xa, Xb = X.copy(), X.copy()
                Xa[i, k] += hh
                Xb[i, k] -= hh
                return (p.loss(Xa, y, None, s, m, **kw).L - p.loss(Xb, y, None, s, m, **kw).L) / (2 * hh)
            num[i, k] = (4 * D(h / 2) - D(h)) / 3
    np.testing.assert_allclose(r.dx, num, rtol=1e-5, atol=1e-7)


def test_phi_sum_is_occupancy_times_mean_and_max_bounds_mean():
    """Invariants: sum = C_occ * mean (per row); max >= mean; hinge(mean) >= mean."""
    rng = np.random.default_rng(44)
    C, d = 30, 16
    T = rng.standard_normal((C, d)); T /= np.linalg.norm(T, axis=1, keepdims=True)
    p = Pool(C, d, F32)
    p.enqueue(T[:20].astype(np.float32), rng.integers(0, 10, 20))   # partially filled
    X = rng.standard_normal((8, d)).astype(np.float32)
    y = np.arange(100, 108)
    mean = p.loss(X, y, None, 30.0, 0.3).phi
    sm = p.loss(X, y, None, 30.0, 0.3, phi_mode=PHI_SUM).phi
    mx = p.loss(X, y, None, 30.0, 0.3, phi_mode=PHI_MAX).phi
    hm = p.loss(X, y, None, 30.0, 0.3, hinge=True).phi
    np.testing.assert_allclose(sm, 20 * mean, rtol=1e-12)
    assert np.all(mx >= mean) and np.all(hm >= mean)


# ----------------------------------------------------------------------------- NEXT-3 duplicates
def test_exclude_stale_duplicates_equals_deleting_them():
    """Variant 'exclude stale self-duplicates': for in-pool rows it must equal the D8 loss on
    the pool with the older same-label slots deleted (independent formulation: a smaller pool)."""
    rng = np.random.default_rng(51)
    C, d = 24, 8
    T = rng.standard_normal((C, d)); T /= np.linalg.norm(T, axis=1, keepdims=True)
    lab = rng.integers(0, 6, C)                     # many duplicates
    p = Pool(C, d, F32)
    p.enqueue(T.astype(np.float32), lab)
    y = np.array([0, 1, 2, 3, 4, 5, 2, 0])
    X = rng.standard_normal((len(y), d)).astype(np.float32)
    r = p.loss(X, y, None, 20.0, 0.3, excl_dup=True)
    assert r.N_neg == 0
    for i in range(len(y)):
        keep = [c for c in range(C) if lab[c] != y[i] or c == r.tslot[i]]   # newest one of y_i stays
        q = Pool(len(keep), d, F32)
        q.enqueue(T[keep].astype(np.float32), lab[keep])
        ri = q.loss(X[i:i + 1], y[i:i + 1], None, 20.0, 0.3)
        assert r.ell[i] == pytest.approx(ri.ell[0], rel=1e-12)
        # per-row gradient scales with 1/N_pos: compare the row's own gradient
        np.testing.assert_allclose(r.dx[i] * len(y), ri.dx[0], rtol=1e-10, atol=1e-13)


def test_exclude_stale_duplicates_closed_form_and_out_of_pool():
    """SURVEY case F pool [(.8,.6) lab 7 older, (0,1) lab 3, (1,0) lab 7 newest, (.6,.8) lab 5]:
    with the stale (.8,.6) excluded the row x=(0,1), y=7 sees {(0,1), (1,0)t, (.6,.8)}:
    L = log(e^{s*1} + e^{s*(0-m)} + e^{s*.8}) - s*(0-m); out-of-pool rows are unchanged."""
    p = _pool_from([([0.8, 0.6], 7), ([0.0, 1.0], 3), ([1.0, 0.0], 7), ([0.6, 0.8], 5)])
    s, m = 64.0, 0.35
    r = p.loss(np.array([[0.0, 1.0]], np.float32), np.array([7]), None, s, m, excl_dup=True)
    z = np.array([s * 1.0, s * (0.0 - m), s * np.float64(np.float32(0.8))])
    want = np.log(np.exp(z - z.max()).sum()) + z.max() - s * (0.0 - m)
    assert r.L == pytest.approx(want, rel=1e-9)
    X = np.array([[0.3, 0.7], [0.9, -0.2]], np.float32)
    a = p.loss(X, np.array([99, 98]), None, s, m, excl_dup=True)
    b = p.loss(X, np.array([99, 98]), None, s, m)
    assert a.L == b.L and np.array_equal(a.dx, b.dx)


# ----------------------------------------------------------------------------- NEXT-3 refresh-in-place enqueue
def _queue_refresh(q, ids, feats, C):
    """SPEC's insert_batch as a literal queue: a Python list of [id, feat],
    oldest first.  Resident ids (their newest entry) are refreshed in place, new ids are
    appended in block order, the overflow is dropped from the front.  Reading R7: a block id
    that this drops is appended as a new one too, until every block id survives
    (S:307).  Returns the new queue and the number of appended rows."""
    M = len(ids)
    S = set(j for j in range(M) if all(e[0] != ids[j] for e in q))
    while True:
        q2 = [list(e) for e in q]
        for j in range(M):
            if j in S:
                continue
            for e in reversed(q2):          # the newest entry of the id (D8)
                if e[0] == ids[j]:
                    e[1] = feats[j]
                    break
        for j in range(M):
            if j in S:
                q2.append([ids[j], feats[j]])
        q2 = q2[-C:]
        alive = [e[0] for e in q2]
        missing = set(j for j in range(M) if ids[j] not in alive
                      or [e for e in q2 if e[0] == ids[j]][-1][1] != feats[j])
        if not missing:
            return q2, len(S)
        S |= missing


def _ring_in_order(p):
    E, C = int(p.E[0]), p.C
    order = np.arange(E) if E < C else (np.arange(C) + E) % C
    return [[int(p.lab[c]), float(p.T[c, 0])] for c in order]


def test_refresh_spec_examples():
    """S:280 'a resident identity re-inserted -> fill_count unchanged, features replaced';
    S:278's FIFO when nothing is resident; reading R7 when the resident is the oldest."""
    p = Pool(4, 1, F32)
    p.enqueue(np.array([[1.0], [2.0]], np.float32), np.array([10, 20]), refresh=True)
    p.enqueue(np.array([[1.5]], np.float32), np.array([10]), refresh=True)     # not full
    assert int(p.E[0]) == 2 and p.lab[:2].tolist() == [10, 20] and p.T[0, 0] == 1.5
    assert p.blk_seq.tolist() == [0]
    for blk in ([3, 4], [5, 6]):
        q = Pool(4, 1, F32)
        q.enqueue(np.array([[1], [2]], np.float32), np.array([1, 2]), refresh=True)
        q.enqueue(np.array([[3], [4]], np.float32), np.array([3, 4]), refresh=True)
        q.enqueue(np.array([[5], [6]], np.float32), np.array([5, 6]), refresh=True)
        assert q.lab.tolist() == [5, 6, 3, 4]
    # full pool A,B,C,D (A oldest): re-insert C with new G -> C refreshed in place (age kept),
    # G takes A's slot
    p = Pool(4, 1, F32)
    p.enqueue(np.array([[1], [2], [3], [4]], np.float32), np.array([1, 2, 3, 4]), refresh=True)
    p.enqueue(np.array([[3.5], [7]], np.float32), np.array([3, 7]), refresh=True)
    assert p.lab.tolist() == [7, 2, 3, 4] and p.T[2, 0] == 3.5 and int(p.E[0]) == 5
    assert p.blk_seq.tolist() == [2, 4]
    # re-insert A (the oldest) with new E: E's append evicts A, so A is appended too (R7)
    p = Pool(4, 1, F32)
    p.enqueue(np.array([[1], [2], [3], [4]], np.float32), np.array([1, 2, 3, 4]), refresh=True)
    p.enqueue(np.array([[1.5], [5]], np.float32), np.array([1, 5]), refresh=True)
    assert p.lab.tolist() == [1, 5, 3, 4] and p.T[0, 0] == 1.5 and int(p.E[0]) == 6
    assert [int(v) for v in p.blk_seq] == [4, 5]
    with pytest.raises(oracle.OracleError):
        p.enqueue(np.array([[1], [2]], np.float32), np.array([9, 9]), refresh=True)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_refresh_equals_queue_model_random(seed):
    """The ring under refresh-in-place equals the literal queue model above after many random
    blocks (labels from a small range, so residency and evictions of residents are common),
    also starting from a pool with duplicates made by pure Eq. 7 enqueues."""
    rng = np.random.default_rng(seed)
    C = int(rng.integers(3, 40))
    p = Pool(C, 1, F32)
    q = []
    n_lab = max(2, C // 2 + int(rng.integers(0, C)))
    for it in range(300):
        M = int(rng.integers(1, min(C, n_lab) + 1))
        ids = rng.choice(n_lab, size=M, replace=False).astype(np.int64)
        feats = (rng.integers(1, 10**6, M) + it * 10**6).astype(np.float32)[:, None]
        if it < 3 and seed == 2:   # pure enqueues first: duplicates in the pool
            p.enqueue(feats, ids)
            q = (q + [[int(a), float(b)] for a, b in zip(ids, feats[:, 0])])[-C:]
            continue
        E0 = int(p.E[0])
        p.enqueue(feats, ids, refresh=True)
        q, n_app = _queue_refresh(q, [int(v) for v in ids], [float(v) for v in feats[:, 0]], C)
        assert int(p.E[0]) - E0 == n_app
        assert _ring_in_order(p) == q
        # every block id is resident with this block's feature, at the slot blk_seq names
        for j in range(M):
            c = int(p.blk_seq[j]) % C
            assert p.lab[c] == ids[j] and p.T[c, 0] == feats[j, 0]


def test_refresh_keeps_age_and_pairing():
    """A refreshed identity keeps its queue position (S:317 'without resetting age'): it is
    evicted at the same step as without the refresh.  The pairing check follows blk_seq."""
    C, M = 8, 2
    p = Pool(C, 1, F32)
    for k in range(4):
        p.enqueue(np.array([[k * 2], [k * 2 + 1]], np.float32), np.array([k * 2, k * 2 + 1]), refresh=True)
    # refresh id 4 (written at step 2) at step 4, then watch when it leaves
    p.enqueue(np.array([[44.0], [100.0]], np.float32), np.array([4, 100]), refresh=True)
    X = np.array([[44.0]], np.float32)
    r = p.loss(X, np.array([4]), np.array([0], np.int32), 1.0, 0.0)
    assert r.tslot[0] == 4 % C and r.N_pos == 1
    with pytest.raises(oracle.OracleError):
        p.loss(X, np.array([4]), np.array([1], np.int32), 1.0, 0.0)
    gone = None
    for k in range(5, 9):
        p.enqueue(np.array([[200.0 + k], [300.0 + k]], np.float32), np.array([200 + k, 300 + k]), refresh=True)
        if 4 not in p.lab.tolist() and gone is None:
            gone = k
    assert gone == 6   # written at step 2 (positions 4,5), evicted when positions 12,13 are written
