"""Wall time of the degree-2 multilevel correction (informational)."""
import sys
import time
sys.path.insert(0, ".")
import paper_1401_4969_b200 as mlg

for L in (3, 4, 5):
    cfg = mlg.RunConfig(domain=mlg.DomainRect(0.0, 1.0, 0.0, 1.0), H=1 / 16, delta=1 / 16, m=16,
                        n_levels=L, nev=1, degree=2)
    with mlg.Hierarchy(cfg) as hy:
        hy.extend_to(L)
        t = time.time()
        lam, pairs, matched, times = mlg.multilevel_correction(hy)
        el = time.time() - t
        tl = times[-1]
        print(f"P2 L{L}: ndofs_int={hy.level_info(L).n_interior} total {el:.3f}s last step "
              f"local {tl.local_seconds:.3f} iface {tl.iface_seconds:.3f} aug {tl.aug_seconds:.4f} "
              f"its {tl.local_iterations_max}/{tl.strip_iterations_max} lam {lam[-1][0]:.12f}",
              flush=True)
