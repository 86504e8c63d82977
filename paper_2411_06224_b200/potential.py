"""IncrementalPotential on the device (solver/incremental_potential.hpp:19-405):
the caller of the hot path that turns a state into its gradient and reduced
block Hessian, composed from the C-ABI entry points with every array resident
in HBM — contact-node positions (node_displacements), the broad phase
(adipc_gpu_broad_phase_device), the contact node stream
(adipc_gpu_contact_emit_device), the inertia / element / body stream
(adipc_gpu_fem_emit_device), the gradient lift and the two-level reduction +
filter + sort + reduce into the context's matrix
(adipc_gpu_assemble_contact_device). Same method names and meaning as the
reference class; the state is the block-numbered vector [x; q] (the layout
newton.hpp's apply_direction works on)."""
from __future__ import annotations

import torch

from .context import Context, InvalidArgument


class IncrementalPotential:
    """mesh: Context.fem_emit's mesh dict (device tensors; an optional
    "bodies" entry holds reduced_mass / kappa / volume — q and q_tilde come
    from the state and set_targets); surface: device int32 tensors verts /
    edges / tris of the ContactSurface (contact-node ids); dofs: the DofMap —
    n_fem and the device tensors abd_body (body of each affine-body contact
    node) and jac36 (its 3 x 12 column-major Jacobian); pinned: device uint8
    per block slot (the constructor's slot_pinned_, :21-31)."""

    def __init__(self, ctx: Context, mesh: dict, surface: dict, dofs: dict, dt: float, pinned=None):
        self.ctx, self.mesh, self.surf, self.dofs = ctx, dict(mesh), surface, dofs
        self.dt2 = float(dt) * float(dt)
        self.n_fem = int(dofs["n_fem"])
        self.n_verts = int(mesh["mass"].numel())
        if self.n_verts != self.n_fem:
            raise InvalidArgument("mesh vertices and DofMap FEM slots differ")
        b = mesh.get("bodies")
        self.n_bodies = 0 if b is None else int(b["kappa"].numel())
        self.n_blocks = self.n_fem + 4 * self.n_bodies
        self.abd_body, self.jac36 = dofs.get("abd_body"), dofs.get("jac36")
        self.n_nodes = self.n_fem + (0 if self.abd_body is None else self.abd_body.numel())
        self.pinned = pinned
        self.dev = mesh["mass"].device
        self.dhat = self.kappa = 0.0
        self.ground = None
        self.friction = None
        self.x_tilde = self.q_tilde = None
        self.last = {}
        self.profile = False  # CUDA-event phase times of assemble() into self.last["phase_ms"]

    # -- configuration (:34-59) ----------------------------------------------
    def set_targets(self, x_tilde, q_tilde=None):
        self.x_tilde, self.q_tilde = x_tilde, q_tilde

    def set_contact(self, dhat: float, kappa: float):
        self.dhat, self.kappa = float(dhat), float(kappa)

    def set_ground(self, normal, height: float):
        """Scene::ground (the contact surface's vertices against a plane)."""
        self.ground = (tuple(float(v) for v in normal), float(height))

    def set_friction(self, constraints: dict, mu: float, eps: float):
        """constraints: device fr_nodes / fr_n / fr_coeff / fr_t1 / fr_t2 /
        fr_lambda and fr_base (the contact-node positions at the step start)."""
        self.friction = dict(constraints, mu=float(mu), fr_eps=float(eps))

    def clear_friction(self):
        self.friction = None

    def begin_friction(self, state, mu: float, eps: float):
        """The step-start freeze of newton.hpp:104-113: friction constraints
        from the contacts at `state` (build_friction_constraints,
        friction.hpp:95-149: proximity broad phase, contact frames, tangent
        bases, lagged normal forces) with the positions as the base; returns
        the number of constraints."""
        pos = self.contact_positions(state)
        pt, ee = self.candidates(pos)
        fr = self.ctx.friction_constraints({"pos": pos, "pt": pt, "ee": ee, "dhat": self.dhat, "kappa": self.kappa,
                                            "ground": self.ground, "surf_verts": self.surf["verts"]})
        fr["fr_base"] = pos.clone()
        self.set_friction(fr, mu, eps)
        return int(fr["fr_n"].numel())

    # -- helpers ----------------------------------------------------------------
    def _split(self, state):
        if not state.is_cuda or state.numel() != 3 * self.n_blocks:
            raise InvalidArgument(f"state: device tensor of 3 * n_blocks = {3 * self.n_blocks} doubles expected")
        return state[: 3 * self.n_fem], state[3 * self.n_fem:]

    def _mesh(self, q):
        m = dict(self.mesh)
        if self.n_bodies:
            m["bodies"] = dict(self.mesh["bodies"], q=q, q_tilde=self.q_tilde)
        return m

    def contact_positions(self, state):
        """contact_node_positions (scene.hpp:112-120): FEM x, affine-body nodes
        A x_bar + p in the reference's operation order."""
        pos = torch.empty(3 * self.n_nodes, dtype=torch.float64, device=self.dev)
        self.ctx.contact_positions(state, self.n_fem, self.abd_body, self.jac36, pos)
        return pos

    def candidates(self, pos, disp=None, inflate=None):
        """proximity_candidates / find_candidates (broad_phase.hpp:143-211):
        node stencils (pt, ee) as device int32 k x 4 tensors."""
        _, pt, _, ee = self.ctx.broad_phase(pos, self.surf["verts"], self.surf["edges"], self.surf["tris"],
                                            self.dhat if inflate is None else inflate, disp=disp)
        return pt, ee

    def _contact(self, pos, pt, ee):
        c = {"pos": pos, "pt": pt, "ee": ee, "dhat": self.dhat, "kappa": self.kappa, "ground": self.ground,
             "surf_verts": self.surf["verts"]}
        if self.friction is not None:
            c.update(self.friction)
        return c

    # -- the reference's methods ---------------------------------------------
    def value(self, state) -> float:
        """:61-159 — inertia + elastic + bodies + barrier / ground / friction
        (+inf once a stencil touches)."""
        x, q = self._split(state)
        v = self.ctx.fem_value(self._mesh(q), x, self.x_tilde, self.dt2, pinned=self.pinned)
        if self.dhat > 0:
            pos = self.contact_positions(state)
            pt, ee = self.candidates(pos)
            v += self.ctx.contact_value(self._contact(pos, pt, ee), self.dt2)
        return v

    def assemble(self, state, project: bool = True):
        """:162-258 — returns (value, grad) with grad a device tensor in block
        numbering; the reduced block Hessian is left in the context (U, the
        two-level tile count and the contact stencil counts in self.last)."""
        x, q = self._split(state)
        mesh = self._mesh(q)
        marks = []

        def mark(name):
            if self.profile:
                e = torch.cuda.Event(enable_timing=True)
                st = self.ctx.stream
                e.record(st if isinstance(st, torch.cuda.Stream) else torch.cuda.current_stream(self.dev))
                marks.append((name, e))

        mark("start")
        nt = int(self.mesh["tets"].numel() // 4)
        cap = self.n_verts + 10 * nt + 20 * self.n_bodies
        sh = self.mesh.get("shells")
        if sh is not None:
            cap += 6 * int(sh["tris"].numel() // 3) + 10 * int(sh["hinges"].numel() // 4)
        keys = torch.empty(cap, dtype=torch.int64, device=self.dev)
        vals = torch.empty((cap, 9), dtype=torch.float64, device=self.dev)
        grad = torch.empty(3 * self.n_blocks, dtype=torch.float64, device=self.dev)
        val = self.ctx.fem_emit(mesh, x, self.x_tilde, self.dt2, keys, vals, grad, project=project,
                                pinned=self.pinned)
        mark("elements")
        n_pt = n_ee = nk = 0
        nkeys = torch.empty(0, dtype=torch.int64, device=self.dev)
        nvals = torch.empty((0, 9), dtype=torch.float64, device=self.dev)
        if self.dhat > 0:
            pos = self.contact_positions(state)
            pt, ee = self.candidates(pos)
            mark("broad_phase")
            n_pt, n_ee = pt.shape[0], ee.shape[0]
            ncap = 10 * (n_pt + n_ee)
            if self.ground is not None:
                ncap += self.surf["verts"].numel()
            if self.friction is not None:
                ncap += 10 * self.friction["fr_n"].numel()
            nkeys = torch.empty(max(ncap, 1), dtype=torch.int64, device=self.dev)
            nvals = torch.empty((max(ncap, 1), 9), dtype=torch.float64, device=self.dev)
            ngrad = torch.empty(3 * self.n_nodes, dtype=torch.float64, device=self.dev)
            cv, nk = self.ctx.contact_emit(self._contact(pos, pt, ee), self.dt2, nkeys, nvals, ngrad,
                                           project=project)
            val += cv
            self.ctx.lift_node_grad(ngrad, self.n_fem, self.abd_body, self.jac36, grad, pinned=self.pinned)
            mark("contact")
        abd_body = self.abd_body if self.abd_body is not None else torch.empty(0, dtype=torch.int32, device=self.dev)
        jac = self.jac36 if self.jac36 is not None else torch.empty(0, dtype=torch.float64, device=self.dev)
        U, n_tiles = self.ctx.assemble_contact(keys, vals, nkeys[:nk], nvals[:nk], self.n_fem, self.n_bodies, abd_body,
                                               jac, self.n_blocks, self.pinned)
        mark("reduce")
        self.last = {"U": U, "contact_tiles": n_tiles, "n_pt": n_pt, "n_ee": n_ee, "node_blocks": nk,
                     "dof_blocks": cap}
        if marks:
            marks[-1][1].synchronize()
            self.last["phase_ms"] = {marks[i + 1][0]: marks[i][1].elapsed_time(marks[i + 1][1])
                                     for i in range(len(marks) - 1)}
        return val, grad

    def ccd_step(self, state, d):
        """contact/ccd.hpp:88-110 over the broad phase of the swept boxes:
        the largest alpha <= 1 the direction d (block numbering) may take."""
        pos = self.contact_positions(state)
        disp = torch.empty_like(pos)
        self.ctx.node_displacements(d, self.n_fem, self.abd_body, self.jac36, disp)
        pt, ee = self.candidates(pos, disp=disp)
        return self.ctx.ccd_step(self._contact(pos, pt, ee), disp)
