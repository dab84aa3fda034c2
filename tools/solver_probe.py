"""C4 solve on the GPU: wall time per iteration and (under ncu) the kernel list.
    python tools/solver_probe.py [max_iters] [bicgstab|gmres]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2409_03095_b200 import generators as G
    from paper_2409_03095_b200 import solvers as S
    from paper_2409_03095_b200.engine import DeviceEngine
    from paper_2409_03095_b200.mcspai import McConfig
    it = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    method = sys.argv[2] if len(sys.argv) > 2 else "bicgstab"
    b = G.convection_diffusion(1000)
    eng = DeviceEngine(0)
    bt = DeviceEngine.upload(b)
    d = eng.build(b.n, *bt, McConfig())
    mt = eng.to_tensors(d)[:3]
    cfg = S.SolverConfig(method=S.SolverMethod[method], rel_tol=1e-6, max_iters=it)
    S.solve_device(b.n, bt, mt, None, cfg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, rep = S.solve_device(b.n, bt, mt, None, cfg)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"iterations {rep.iterations} wall {1e3 * dt:.1f} ms  per-iteration {1e3 * dt / max(rep.iterations, 1):.3f} ms "
          f"device {rep.ms:.1f} ms converged={rep.converged}")


if __name__ == "__main__":
    main()
