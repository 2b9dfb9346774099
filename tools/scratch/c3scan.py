import sys, json
sys.path.insert(0, "/root/repo")
import paper_2309_11488_b200 as P
import paper_2309_11488_b200.synthetic as S
for sig in (1.0, 1.5, 2.0):
    for boost in (1e-2, 1e-3, 1e-4):
        g = S.generate_heterogeneous(92, 224, 17, sigma_k=sig, diagonal_boost=boost)
        out = {"sigma": sig, "boost": boost}
        for be in ("level", "color"):
            cfg = P.SolverConfig(backend=P.Backend.from_name(be), stop=P.StoppingCriteria(1e-8, 400))
            try:
                x, rep = P.solve_with_fallback(cfg, g.a, g.rhs)
                out[be] = (rep.iterations, rep.converged, rep.fallback_used)
            except Exception as e:
                out[be] = repr(e)[:80]
        print(json.dumps(out), flush=True)
