"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container, where the read-only reference is importable:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden.py

It imports ``aqr`` from /root/reference/pkg/src (never copied into this
repo), runs ``aqr.factorize`` on seeded inputs and writes

* tests/golden/small.npz -- inputs and the reference's Q, R, flagged
  columns and mv counts for small dense/CSR instances, every GS method;
* tests/golden/cases.json -- breakdown / flag known-answer results, and for
  config 1 (tests/cfg1.py) the SHA-256 of the inputs, of the reference's Q
  and R per method, the reference's R matrices' digests and its accuracy
  metrics (metrics.py:35-53).

The GPU box never runs this script (/root/reference does not exist there);
it only reads the committed outputs.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

import aqr  # noqa: E402  (the reference package)

import cfg1  # noqa: E402

GS_METHODS = [str(m) for m in aqr.ALL_GS_METHODS]
MGS_METHODS = [m for m in GS_METHODS if m.startswith("mgs")]


def random_instance(seed, m, n):
    """pkg/tests/test_gram_schmidt.py:58-63 recipe."""
    rng = aqr.make_rng(seed)
    G = rng.standard_normal((m, m))
    A = np.asfortranarray(G @ G.T + m * np.eye(m))
    Z = np.asfortranarray(rng.standard_normal((m, n)))
    return Z, A


def run_all(store, key, Z, op, methods):
    for meth in methods:
        try:
            r = aqr.factorize(Z, op, meth)
        except aqr.BreakdownError as e:
            store[f"{key}|{meth}|breakdown"] = np.array([e.column, e.value])
            continue
        store[f"{key}|{meth}|Q"] = r.Q
        store[f"{key}|{meth}|R"] = r.R
        store[f"{key}|{meth}|flag"] = np.array(r.flagged_columns, dtype=np.int64)
        store[f"{key}|{meth}|mv"] = np.array([r.cost.mv_count, r.cost.flops], dtype=np.int64)


def main():
    store = {}
    cases = {}

    # hand instance (test_gram_schmidt.py:66-77)
    Z = np.array([[1.0, 1.0], [0.0, 1.0]], order="F")
    A = np.diag([1.0, 4.0])
    store["hand|Z"], store["hand|A"] = Z, np.asfortranarray(A)
    run_all(store, "hand", Z, aqr.DenseSpdOperator(A), GS_METHODS + ["cholqr"])

    # small dense random instances
    dense = [(0, 5, 1), (1, 12, 4), (2, 25, 7), (3, 40, 13), (7, 64, 64)]
    for seed, m, n in dense:
        key = f"dense{seed}"
        Z, A = random_instance(seed, m, n)
        store[f"{key}|Z"], store[f"{key}|A"] = Z, A
        run_all(store, key, Z, aqr.DenseSpdOperator(A), GS_METHODS + ["cholqr"])

    # A = I against the textbook MGS (test_gram_schmidt.py:133-150)
    Z, _ = random_instance(4, 25, 7)
    store["ident|Z"], store["ident|A"] = Z, np.asfortranarray(np.eye(25))
    run_all(store, "ident", Z, aqr.identity_operator(25), MGS_METHODS)

    # ill-conditioned dense (kappa(A)=1e8, kappa(A^1/2 Z)=1e10, case 2)
    rng = aqr.make_rng(11)
    factors, op = aqr.build_spd(60, 1e8, rng)
    Z = aqr.build_Z(aqr.CaseSpec(2, 60, 12, 1e8, 1e10, 11), factors, rng)
    store["illcond|Z"], store["illcond|A"] = Z, op.matrix
    run_all(store, "illcond", Z, op, GS_METHODS)

    # CSR: the reference's own 5-point Laplacian (testbed.py:128-153)
    for key, (nx, ny, n, seed) in {"csr9x7": (9, 7, 12, 3), "csr16": (16, 16, 8, 5)}.items():
        op = aqr.laplacian_spd(nx, ny)
        Z = np.asfortranarray(np.random.default_rng(seed).standard_normal((op.dim, n)))
        store[f"{key}|Z"] = Z
        store[f"{key}|indptr"], store[f"{key}|indices"], store[f"{key}|data"] = (
            op.indptr, op.indices, op.data)
        run_all(store, key, Z, op, GS_METHODS)

    # known-answer exceptions
    kat = {}
    Zb = np.array([[1.0, 2.0], [0.0, 0.0], [0.0, 0.0]])
    for meth in GS_METHODS:
        try:
            aqr.factorize(Zb, aqr.identity_operator(3), meth)
            kat[meth] = None
        except aqr.BreakdownError as e:
            kat[meth] = [e.column, e.value]
    cases["breakdown_rank_deficient"] = kat
    flag = {}
    for meth in GS_METHODS:
        r = aqr.factorize(np.array([[1.0], [1e-16]]), aqr.diagonal_operator([1e-30, 1.0]), meth)
        flag[meth] = {"flagged": r.flagged_columns, "R00": r.R[0, 0], "Q": r.Q.ravel().tolist()}
    cases["flag_tiny_norm"] = flag

    # config 1: hashes of inputs and the reference outputs, plus metrics
    A, Z = cfg1.make()
    op = aqr.DenseSpdOperator(A)
    c1 = {"A_sha": cfg1.sha(A), "Z_sha": cfg1.sha(Z), "methods": {}}
    for meth in MGS_METHODS + ["cgs-ha-row", "cgs-hp-row", "cgs-naive-row"]:
        r = aqr.factorize(Z, op, meth)
        loss = aqr.loss_of_A_orthogonality(r.Q, op)
        rep_abs, rep_rel = aqr.representation_error(Z, r.Q, r.R)
        c1["methods"][meth] = {
            "Q_sha": cfg1.sha(r.Q), "R_sha": cfg1.sha(r.R), "flagged": r.flagged_columns,
            "mv_count": r.cost.mv_count, "loss_A_orth": loss, "rep_abs": rep_abs,
            "rep_rel": rep_rel, "rep_rel_Z": float(rep_abs / aqr.two_norm(Z)),
            "R_diag": np.diag(r.R).tolist(),
        }
        store[f"cfg1|{meth}|R"] = r.R
    cases["cfg1"] = c1

    np.savez_compressed(os.path.join(HERE, "small.npz"), **store)
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(cases, f, indent=1, sort_keys=True)
    print("wrote", len(store), "arrays")


if __name__ == "__main__":
    main()
