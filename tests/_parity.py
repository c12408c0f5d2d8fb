"""Parity metrics of the north star: eigenvalue relative error,
eigenfunction relative L2 (M-norm) up to sign, and for clusters with relative
gap < 1e-6 the distance of the computed vectors from the oracle subspace."""
import numpy as np

LAMBDA_RTOL = 1e-10
VEC_RTOL = 1e-8


def mnorm_fn(apply_mass, expand):
    def mn(w):
        f = expand(w)
        return float(np.sqrt(max(f @ apply_mass(f), 0.0)))
    return mn


def clusters(lams, gap=1e-6):
    groups, cur = [], [0]
    for i in range(1, len(lams)):
        if abs(lams[i] - lams[cur[-1]]) <= gap * abs(lams[i]):
            cur.append(i)
        else:
            groups.append(cur)
            cur = [i]
    groups.append(cur)
    return groups


def compare_pairs(lam_gpu, vec_gpu, lam_ref, vec_ref, apply_mass, expand,
                  lam_rtol=LAMBDA_RTOL, vec_rtol=VEC_RTOL, gap=1e-6):
    """Returns the worst (lambda rel err, vector rel err).  Eigenvalues closer
    than `gap` (relative) are compared as a subspace."""
    lam_gpu = np.asarray(lam_gpu)
    lam_ref = np.asarray(lam_ref)
    lerr = np.max(np.abs(lam_gpu - lam_ref) / np.abs(lam_ref))
    assert lerr <= lam_rtol, (lam_gpu, lam_ref, lerr)
    mn = mnorm_fn(apply_mass, expand)

    def mdot(a, b):
        return float(expand(a) @ apply_mass(expand(b)))

    verr = 0.0
    for grp in clusters(lam_ref, gap):
        if len(grp) == 1:
            i = grp[0]
            u, v = vec_gpu[i], vec_ref[i]
            s = 1.0 if mdot(u, v) >= 0 else -1.0
            verr = max(verr, mn(u - s * v) / mn(v))
        else:  # subspace distance ||(I - P_ref) u||_M / ||u||_M
            V = [vec_ref[i] / mn(vec_ref[i]) for i in grp]
            G = np.array([[mdot(a, b) for b in V] for a in V])
            L = np.linalg.cholesky(G)
            Linv = np.linalg.inv(L)
            Q = [sum(Linv[r, c] * V[c] for c in range(len(V))) for r in range(len(V))]
            for i in grp:
                u = vec_gpu[i]
                res = u - sum(mdot(q, u) * q for q in Q)
                verr = max(verr, mn(res) / mn(u))
    assert verr <= vec_rtol, verr
    return lerr, verr


# Seeded random-projection sketch (Johnson-Lindenstrauss): for R with iid
# uniform(-1,1) rows, E[(R w)_k^2] = ||w||^2 / 3, so ||S(u - v)|| / ||S v|| estimates
# the full-vector relative l2 difference ||u - v|| / ||v|| (K=32: within a factor
# ~1.3 with high probability).  On the uniform P1 lattice the mass matrix is
# spectrally equivalent to h^2 I, so the
# l2 estimate bounds the M-norm difference of the north star within a factor 2
# (P1 mass stencil h^2/12 * [6; six 1s]: eigenvalues in [h^2/4, h^2]).
SKETCH_K = 32
SKETCH_SEED = 20261020


def sketch(vecs, k=SKETCH_K, seed=SKETCH_SEED):
    """(projections nvec x k, row norms k) of R = uniform(-1,1)[k][n], drawn row by row."""
    vecs = np.atleast_2d(vecs)
    rng = np.random.default_rng(seed)
    proj = np.empty((vecs.shape[0], k))
    rn = np.empty(k)
    for i in range(k):
        r = rng.uniform(-1.0, 1.0, size=vecs.shape[1])
        proj[:, i] = vecs @ r
        rn[i] = np.sqrt(r @ r)
    return proj, rn
