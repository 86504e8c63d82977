"""Small end-to-end drive of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): assembly (plain, filtered,
two-level contact device path), MAS build (solve order and reference
numbering), block Jacobi, preconditioner apply, PCG (graphs + PDL) in the
default and the deterministic mode, SpMV, the post-solve step kernels.
the element-Hessian producer (fast and Jacobi paths) on the cfg1 mesh.
Scenes: the soft cube (cfg1), the stiff beam, the ABD stack (cfg3).
Usage: compute-sanitizer --tool <tool> python tools/sanitize_drive.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_06224_b200 as P  # noqa: E402
import scenegen as scenes  # noqa: E402
from paper_2411_06224_b200 import _lib  # noqa: E402
from paper_2411_06224_b200.context import Context  # noqa: E402

for name in sys.argv[1:] or ["cfg1_soft_cube", "stiff_beam", "cfg3_abd_stack"]:
    sc = scenes.CONFIGS[name]()
    l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
    for det in (0, 1):
        for order in (1, 0):
            c = Context(0)
            c.set_option(_lib.OPT_DETERMINISTIC, det)
            c.set_option(_lib.OPT_SOLVE_ORDER, order)
            c.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
            if sc.n_bodies:
                U, nt = c.assemble_contact(sc.keys, sc.vals, sc.node_keys, sc.node_vals, sc.n_fem, sc.n_bodies,
                                           sc.abd_body, sc.jac36, sc.n_blocks, sc.pinned)
                b = c.spmv(np.random.default_rng(5).standard_normal(3 * sc.n_blocks))
            else:
                c.assemble_filtered(sc.keys, sc.vals, sc.n_blocks, sc.pinned)
                b = scenes.gravity_rhs(sc)
            for kind in (_lib.PRECOND_MAS, _lib.PRECOND_JACOBI):
                c.build_preconditioner(kind)
                z = c.precond_apply(b)
                x, r = c.pcg(b, 1e-4, 50, 100000)
                print(name, "det", det, "order", order, "kind", kind, r, float(np.linalg.norm(z)), flush=True)
            d = torch.from_numpy(x).cuda()
            st = torch.zeros_like(d)
            torch.cuda.synchronize()
            c.step_inf_norm(d, sc.n_fem, 0) if sc.n_bodies == 0 else None
            c.apply_direction(st, d, 0.5, torch.empty_like(d))
            torch.cuda.synchronize()
            c.close()
# the element-Hessian producer: at rest (PSD fast path) and deformed (Jacobi)
sc = scenes.CONFIGS["cfg1_soft_cube"]()
inv9, vol = scenes.tet_rest_data(sc.verts, sc.tets)
mesh = {"mass": torch.from_numpy(sc.mass).cuda(), "tets": torch.from_numpy(sc.tets).cuda(),
        "rest_inv9": torch.from_numpy(inv9).cuda(), "rest_volume": torch.from_numpy(vol).cuda(),
        "tet_begin": [0, len(sc.tets)], "mu": [sc.mu], "lam": [sc.lam]}
c = Context(0)
xt = torch.from_numpy(scenes.inertial_target(sc)).cuda()
pin = torch.from_numpy(sc.pinned).cuda()
for scale in (0.0, 0.3):
    x = sc.verts + np.random.default_rng(1).uniform(-scale, scale, sc.verts.shape) * 0.01
    dx = torch.from_numpy(np.ascontiguousarray(x.reshape(-1))).cuda()
    g = torch.empty_like(dx)
    val, U = c.fem_assemble(mesh, dx, xt, 1e-4, g, pinned=pin)
    print("fem_assemble", scale, val, U, flush=True)
c.close()
# the device IncrementalPotential on a small geometric hybrid scene: positions,
# broad phase (proximity and swept), contact / element / body producers, the
# gradient lift, two-level assembly, line-search value, CCD, cold MAS + PCG
from paper_2411_06224_b200.potential import IncrementalPotential  # noqa: E402
from scenegen.geom import GeomHybrid  # noqa: E402

g = GeomHybrid(grid=(2, 2, 1), res=4, bodies=(2, 2), body_res=1)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
c = Context(0)
l0 = P.partition_block_graph(g.n_blocks, g.rest_edges, 16)
c.set_level0_partition(l0.part_of, l0.n_parts, 16, 4)
mesh = {"mass": t(g.mass), "tets": t(g.tets), "rest_inv9": t(g.rest_inv9), "rest_volume": t(g.rest_volume),
        "tet_begin": g.tet_begin, "mu": [g.mu], "lam": [g.lam],
        "bodies": {"reduced_mass": t(g.reduced_mass.transpose(0, 2, 1)), "kappa": t(g.kappa_abd),
                   "volume": t(g.body_volume)}}
ip = IncrementalPotential(c, mesh, {"verts": t(g.surf_verts), "edges": t(g.edges), "tris": t(g.tris)},
                          {"n_fem": g.n_fem, "abd_body": t(g.abd_body), "jac36": t(g.jac36)}, g.dt, pinned=t(g.pinned))
ip.set_targets(t(g.x_tilde.reshape(-1)), t(g.q_tilde))
ip.set_contact(g.dhat, g.kappa)
state = t(g.state() + np.random.default_rng(2).normal(0, 5e-5, 3 * g.n_blocks))
val, grad = ip.assemble(state)
print("potential", val, ip.last, ip.value(state), flush=True)
c.build_preconditioner(_lib.PRECOND_MAS)
d = torch.empty_like(grad)
_, res = c.pcg(-grad, 1e-4, 250, 100000, x=d)
print("ccd", ip.ccd_step(state, d), res, flush=True)
c.close()
print("sanitize drive done")
