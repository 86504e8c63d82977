"""Per-scene device context over the C-ABI (include/adipc_gpu.h).

A Context owns one device-resident SortedSymBlockCoo, its preconditioner and
the PCG workspace. Array arguments may be numpy arrays (host; the library
copies) or torch CUDA tensors (device; the `_device` entry points are used and
nothing is copied). Status codes are mapped back to the reference's
exceptions: invalid_argument -> InvalidArgument (a ValueError),
indefinite subdomain -> IndefiniteSubdomain (a RuntimeError).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import ptr


class AdipcError(RuntimeError):
    pass


class InvalidArgument(AdipcError, ValueError):
    """std::invalid_argument of the reference (e.g. reduction.hpp:34)."""


class IndefiniteSubdomain(AdipcError):
    """std::runtime_error of mas.hpp:74-77."""


class CudaFailure(AdipcError):
    pass


def _is_device(a) -> bool:
    return a is not None and not isinstance(a, np.ndarray) and getattr(a, "is_cuda", False)


def _raise(rc: int, msg: str):
    if rc == _lib.INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == _lib.INDEFINITE:
        raise IndefiniteSubdomain(msg)
    raise CudaFailure(msg)


class PcgResult:
    """solver/pcg.hpp:10-14."""

    def __init__(self, iters=0, rel_residual=0.0, converged=False):
        self.iters = iters
        self.rel_residual = rel_residual
        self.converged = converged

    def __repr__(self):
        return f"PcgResult(iters={self.iters}, rel_residual={self.rel_residual:.3e}, converged={self.converged})"


class Context:
    def __init__(self, device: int = 0, stream=None):
        self._L = _lib.gpu()
        h = C.c_void_p()
        rc = self._L.adipc_gpu_create(device, C.byref(h))
        if rc != 0:
            _raise(rc, self._L.adipc_gpu_last_error(None).decode())
        self.h = h
        self.device = device
        self.stream = None
        if stream is not None:
            self.set_stream(stream)

    def close(self):
        if getattr(self, "h", None):
            self._L.adipc_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            _raise(rc, self._L.adipc_gpu_last_error(self.h).decode())

    # -- plumbing --------------------------------------------------------------
    def set_stream(self, stream):
        """stream: a torch.cuda.Stream, a raw cudaStream_t int, or None."""
        raw = getattr(stream, "cuda_stream", stream)
        self._check(self._L.adipc_gpu_set_stream(self.h, raw))
        self.stream = stream

    def set_option(self, option: int, value: int):
        self._check(self._L.adipc_gpu_set_option(self.h, option, value))

    def timings(self):
        t = np.zeros(4, np.float32)
        self._check(self._L.adipc_gpu_last_timings(self.h, t))
        return dict(assemble_ms=float(t[0]), build_ms=float(t[1]), build_host_ms=float(t[2]), pcg_ms=float(t[3]))

    def pcg_profile(self):
        t = np.zeros(4, np.float32)
        it = C.c_int()
        self._check(self._L.adipc_gpu_pcg_profile(self.h, t, C.byref(it)))
        return dict(spmv_ms=float(t[0]), update_ms=float(t[1]), precond_ms=float(t[2]), final_ms=float(t[3]),
                    iters=it.value)

    @staticmethod
    def kernel_launches() -> int:
        return int(_lib.gpu().adipc_gpu_kernel_launches())

    # -- assembly ------------------------------------------------------------------
    def assemble(self, keys, vals, n_block_rows: int, deterministic: bool = True) -> int:
        """sort_stream + fast_hash_reduction into the context matrix; returns U."""
        U = C.c_int64()
        T = len(keys)
        if _is_device(keys):
            self._check(self._L.adipc_gpu_assemble_device(self.h, ptr(keys), ptr(vals), T, n_block_rows,
                                                          int(deterministic), C.byref(U)))
        else:
            k = np.ascontiguousarray(keys, np.uint64)
            v = np.ascontiguousarray(vals, np.float64).reshape(-1, 9)
            self._check(self._L.adipc_gpu_assemble(self.h, ptr(k), ptr(v), T, n_block_rows, int(deterministic),
                                                   C.byref(U)))
        return U.value

    def assemble_filtered(self, keys, vals, n_block_rows: int, pinned, deterministic: bool = True) -> int:
        """filter_pinned + sort_stream + fast_hash_reduction (incremental_potential.hpp:255-257)."""
        U = C.c_int64()
        T = len(keys)
        if _is_device(keys):
            self._check(self._L.adipc_gpu_assemble_filtered_device(self.h, ptr(keys), ptr(vals), T, n_block_rows,
                                                                   ptr(pinned), int(deterministic), C.byref(U)))
        else:
            k = np.ascontiguousarray(keys, np.uint64)
            v = np.ascontiguousarray(vals, np.float64).reshape(-1, 9)
            p = np.ascontiguousarray(pinned, np.uint8)
            self._check(self._L.adipc_gpu_assemble_filtered(self.h, ptr(k), ptr(v), T, n_block_rows, ptr(p),
                                                            int(deterministic), C.byref(U)))
        return U.value

    def assemble_contact(self, keys, vals, node_keys, node_vals, n_fem, n_bodies, abd_node_body, jac36,
                         n_block_rows: int, pinned=None):
        """two_level_abd_reduce + append + filter_pinned + sort + reduce
        (incremental_potential.hpp:392-394, 253-257) in one call; the reduced
        contact tiles stay on the device. Returns (U, n_tiles)."""
        U, nt = C.c_int64(), C.c_int64()
        T, Tn = len(keys), len(node_keys)
        if _is_device(keys):
            self._check(self._L.adipc_gpu_assemble_contact_device(
                self.h, ptr(keys), ptr(vals), T, ptr(node_keys), ptr(node_vals), Tn, n_fem, n_bodies,
                len(abd_node_body), ptr(abd_node_body), ptr(jac36), n_block_rows, ptr(pinned), C.byref(U),
                C.byref(nt)))
        else:
            k = np.ascontiguousarray(keys, np.uint64)
            v = np.ascontiguousarray(vals, np.float64).reshape(-1, 9)
            nk = np.ascontiguousarray(node_keys, np.uint64)
            nv = np.ascontiguousarray(node_vals, np.float64).reshape(-1, 9)
            body = np.ascontiguousarray(abd_node_body, np.int32)
            jac = np.ascontiguousarray(jac36, np.float64).reshape(-1, 36)
            p = None if pinned is None else np.ascontiguousarray(pinned, np.uint8)
            if p is not None and len(p) != n_block_rows:
                raise InvalidArgument("pinned: one byte per block row expected")
            self._check(self._L.adipc_gpu_assemble_contact(
                self.h, ptr(k), ptr(v), T, ptr(nk), ptr(nv), Tn, n_fem, n_bodies, len(body), ptr(body), ptr(jac),
                n_block_rows, ptr(p), C.byref(U), C.byref(nt)))
        return U.value, nt.value

    # -- element-Hessian producer ------------------------------
    def _fem_desc(self, mesh, x, x_tilde, dt2, project, pinned):
        """mesh: dict of DEVICE tensors mass / tets / rest_inv9 / rest_volume and
        host lists tet_begin / mu / lam (one entry per solid mesh)."""
        tb = np.ascontiguousarray(mesh["tet_begin"], np.int64)
        mu = np.ascontiguousarray(mesh["mu"], np.float64)
        lam = np.ascontiguousarray(mesh["lam"], np.float64)
        n = int(mesh["mass"].numel())
        for name, t in (("x", x), ("x_tilde", x_tilde)):
            if not _is_device(t) or t.numel() != 3 * n:
                raise InvalidArgument(f"{name}: device tensor of 3 * n_verts = {3 * n} doubles expected")
        d = _lib.FemDesc(n, ptr(x), ptr(x_tilde), ptr(mesh["mass"]), len(tb) - 1, tb.ctypes.data, mu.ctypes.data,
                         lam.ctypes.data, ptr(mesh["tets"]), ptr(mesh["rest_inv9"]), ptr(mesh["rest_volume"]),
                         float(dt2), int(project), ptr(pinned) if pinned is not None else None)
        sh = mesh.get("shells")  # device tris / tri_rest / hinges / hinge_rest; host tri_begin / hinge_begin / material
        keep = [tb, mu, lam]
        if sh is not None:
            stb = np.ascontiguousarray(sh["tri_begin"], np.int64)
            shb = np.ascontiguousarray(sh["hinge_begin"], np.int64)
            smat = np.ascontiguousarray(sh["material"], np.float64).reshape(-1)
            kinds = np.ascontiguousarray(mesh["mesh_kind"], np.int32)
            keep += [stb, shb, smat, kinds]
            d.n_shells = len(stb) - 1
            d.tri_begin, d.hinge_begin, d.shell_material = stb.ctypes.data, shb.ctypes.data, smat.ctypes.data
            d.tris, d.tri_rest = ptr(sh["tris"]), ptr(sh["tri_rest"])
            d.hinges, d.hinge_rest = ptr(sh["hinges"]), ptr(sh["hinge_rest"])
            d.n_kinds, d.mesh_kind = len(kinds), kinds.ctypes.data
        b = mesh.get("bodies")  # device tensors q / q_tilde (nb x 12), reduced_mass (nb x 144), kappa, volume
        if b is not None:
            d.n_bodies = int(b["kappa"].numel())
            d.q, d.q_tilde, d.reduced_mass = ptr(b["q"]), ptr(b["q_tilde"]), ptr(b["reduced_mass"])
            d.body_kappa, d.body_volume = ptr(b["kappa"]), ptr(b["volume"])
        return d, keep, n

    def fem_emit(self, mesh, x, x_tilde, dt2, keys, vals, grad, project=True, pinned=None):
        """IncrementalPotential::assemble's inertia + tet stencils into the
        device stream (keys / vals, n + 10 n_tets entries) and grad; returns
        the value."""
        d, keep, _ = self._fem_desc(mesh, x, x_tilde, dt2, project, pinned)
        v = C.c_double()
        self._check(self._L.adipc_gpu_fem_emit_device(self.h, C.byref(d), ptr(keys), ptr(vals), ptr(grad),
                                                      C.byref(v)))
        return v.value

    def fem_value(self, mesh, x, x_tilde, dt2, grad=None, pinned=None):
        """IncrementalPotential::value's inertia + elastic + body terms (the
        line search); optionally the gradient."""
        d, keep, _ = self._fem_desc(mesh, x, x_tilde, dt2, False, pinned)
        v = C.c_double()
        self._check(self._L.adipc_gpu_fem_value_device(self.h, C.byref(d), ptr(grad), C.byref(v)))
        return v.value

    def fem_assemble(self, mesh, x, x_tilde, dt2, grad, project=True, pinned=None):
        """emit + filter_pinned + sort + reduce into the context matrix; returns
        (value, U)."""
        d, keep, _ = self._fem_desc(mesh, x, x_tilde, dt2, project, pinned)
        v, U = C.c_double(), C.c_int64()
        self._check(self._L.adipc_gpu_fem_assemble_device(self.h, C.byref(d), ptr(grad), C.byref(v), C.byref(U)))
        return v.value, U.value

    # -- contact producers ------------------------------------
    @staticmethod
    def contact_desc(c):
        """c: dict of DEVICE tensors pos (n x 3 / 3n), pt / ee (k x 4 int32),
        surf_verts (int32), friction arrays fr_nodes / fr_n / fr_coeff / fr_t1 /
        fr_t2 / fr_lambda / fr_base; scalars dhat, kappa, mu, fr_eps; ground =
        (normal, height) or None."""
        def n_of(name, per=1):
            t = c.get(name)
            return 0 if t is None else t.numel() // per
        d = _lib.ContactDesc()
        d.n_nodes = n_of("pos", 3)
        d.pos = ptr(c["pos"])
        d.n_pt, d.pt = n_of("pt", 4), ptr(c.get("pt")) if n_of("pt", 4) else None
        d.n_ee, d.ee = n_of("ee", 4), ptr(c.get("ee")) if n_of("ee", 4) else None
        d.dhat, d.kappa = float(c["dhat"]), float(c["kappa"])
        g = c.get("ground")
        d.ground = int(g is not None)
        if g is not None:
            for k in range(3):
                d.ground_normal[k] = float(g[0][k])
            d.ground_height = float(g[1])
        d.n_surf_verts = n_of("surf_verts") if g is not None else 0
        d.surf_verts = ptr(c.get("surf_verts")) if d.n_surf_verts else None
        d.n_friction = n_of("fr_n")
        if d.n_friction:
            for f in ("fr_nodes", "fr_coeff", "fr_t1", "fr_t2", "fr_lambda", "fr_base"):
                setattr(d, f, ptr(c[f]))
            d.fr_n_nodes = ptr(c["fr_n"])
        d.mu, d.fr_eps = float(c.get("mu", 0.0)), float(c.get("fr_eps", 1.0))
        return d

    def contact_emit(self, c, dt2, keys, vals, node_grad, project=True):
        """assemble_contact's node part into the device node stream; returns
        (value, entries written)."""
        d = self.contact_desc(c)
        v, n = C.c_double(), C.c_int64()
        self._check(self._L.adipc_gpu_contact_emit_device(self.h, C.byref(d), float(dt2), int(project), ptr(keys),
                                                          ptr(vals), keys.numel(), ptr(node_grad), C.byref(v),
                                                          C.byref(n)))
        return v.value, n.value

    def lift_node_grad(self, node_grad, n_fem, abd_body, jac36, grad, pinned=None):
        """grad += the contact node gradient (FEM nodes; J^T for body nodes),
        incremental_potential.hpp:395-403 (device tensors); pinned slots get
        nothing."""
        n_abd = 0 if abd_body is None else abd_body.numel()
        self._check(self._L.adipc_gpu_lift_node_grad_device(self.h, ptr(node_grad), n_fem, n_abd, ptr(abd_body),
                                                            ptr(jac36), ptr(pinned), ptr(grad)))

    def broad_phase(self, pos, verts, edges, tris, inflate, disp=None):
        """find_candidates (broad_phase.hpp:143-211) on device tensors; returns
        device int32 tensors (pt_pairs k x 2, pt_stencils k x 4, ee_pairs,
        ee_stencils)."""
        import torch

        npt, nee = C.c_int64(), C.c_int64()
        self._check(self._L.adipc_gpu_broad_phase_device(self.h, pos.numel() // 3, ptr(pos), ptr(disp), verts.numel(),
                                                         ptr(verts), edges.numel() // 2, ptr(edges), tris.numel() // 3,
                                                         ptr(tris), float(inflate), C.byref(npt), C.byref(nee)))
        dev = pos.device
        out = [torch.empty((npt.value, 2), dtype=torch.int32, device=dev),
               torch.empty((npt.value, 4), dtype=torch.int32, device=dev),
               torch.empty((nee.value, 2), dtype=torch.int32, device=dev),
               torch.empty((nee.value, 4), dtype=torch.int32, device=dev)]
        self._check(self._L.adipc_gpu_broad_phase_copy(self.h, *[ptr(t) if t.numel() else None for t in out]))
        return out

    def contact_value(self, c, dt2):
        d = self.contact_desc(c)
        v = C.c_double()
        self._check(self._L.adipc_gpu_contact_value_device(self.h, C.byref(d), float(dt2), C.byref(v)))
        return v.value

    def friction_constraints(self, c):
        """build_friction_constraints (friction.hpp:95-149) over the stencils
        of c (see contact_desc; the friction entries of c are ignored) ->
        dict of device tensors fr_nodes / fr_n / fr_coeff / fr_t1 / fr_t2 /
        fr_lambda in contact_desc's friction format."""
        import torch

        d = self.contact_desc(dict(c, fr_n=None))
        cap = max(d.n_pt + d.n_ee + d.n_surf_verts, 1)
        dev = c["pos"].device
        out = {"fr_nodes": torch.empty((cap, 4), dtype=torch.int32, device=dev),
               "fr_n": torch.empty(cap, dtype=torch.int32, device=dev),
               "fr_coeff": torch.empty((cap, 4), dtype=torch.float64, device=dev),
               "fr_t1": torch.empty((cap, 3), dtype=torch.float64, device=dev),
               "fr_t2": torch.empty((cap, 3), dtype=torch.float64, device=dev),
               "fr_lambda": torch.empty(cap, dtype=torch.float64, device=dev)}
        k = C.c_int64()
        self._check(self._L.adipc_gpu_friction_constraints_device(self.h, C.byref(d), cap, ptr(out["fr_nodes"]),
                                                                  ptr(out["fr_n"]), ptr(out["fr_coeff"]),
                                                                  ptr(out["fr_t1"]), ptr(out["fr_t2"]),
                                                                  ptr(out["fr_lambda"]), C.byref(k)))
        return {name: t[:k.value] for name, t in out.items()}

    def ccd_step(self, c, disp):
        d = self.contact_desc(c)
        a = C.c_double()
        self._check(self._L.adipc_gpu_ccd_step_device(self.h, C.byref(d), ptr(disp), C.byref(a)))
        return a.value

    def matrix_info(self):
        n, U = C.c_int32(), C.c_int64()
        self._check(self._L.adipc_gpu_matrix_info(self.h, C.byref(n), C.byref(U)))
        return n.value, U.value

    # ---- the step after the solve (newton.hpp:257-290); device tensors ----
    def step_inf_norm(self, d_dir, n_fem, n_bodies, d_max_xbar=None):
        out = C.c_double()
        self._check(self._L.adipc_gpu_step_inf_norm_device(self.h, ptr(d_dir), n_fem, n_bodies, ptr(d_max_xbar),
                                                             C.byref(out)))
        return out.value

    def apply_direction(self, d_state, d_dir, alpha, d_out):
        self._check(self._L.adipc_gpu_apply_direction_device(self.h, ptr(d_state), ptr(d_dir), float(alpha),
                                                               d_state.numel(), ptr(d_out)))

    def contact_positions(self, d_state, n_fem, d_abd_body, d_jac36, d_out):
        """contact_node_positions (scene.hpp:112-120): FEM x, body nodes A x_bar + p."""
        n_abd = 0 if d_abd_body is None else d_abd_body.numel()
        self._check(self._L.adipc_gpu_contact_positions_device(self.h, ptr(d_state), n_fem, n_abd, ptr(d_abd_body),
                                                                 ptr(d_jac36), ptr(d_out)))

    def node_displacements(self, d_dir, n_fem, d_abd_body, d_jac36, d_out):
        n_abd = 0 if d_abd_body is None else d_abd_body.numel()
        self._check(self._L.adipc_gpu_node_displacements_device(self.h, ptr(d_dir), n_fem, n_abd, ptr(d_abd_body),
                                                                  ptr(d_jac36), ptr(d_out)))

    def dump_matrix_binary(self, path):
        """Binary capture of the device matrix (api.load_matrix_binary reads it)."""
        self._check(self._L.adipc_gpu_dump_matrix_binary(self.h, str(path).encode()))

    def dump_block_coo(self, path):
        """srbk_spmv.hpp:52-60 of the device matrix (--dump-hessian text)."""
        self._check(self._L.adipc_gpu_dump_block_coo(self.h, str(path).encode()))

    def copy_matrix(self):
        n, U = self.matrix_info()
        rows = np.empty(U, np.uint32)
        cols = np.empty(U, np.uint32)
        blocks = np.empty((U, 9), np.float64)
        self._check(self._L.adipc_gpu_copy_matrix(self.h, ptr(rows), ptr(cols), ptr(blocks)))
        return n, rows, cols, blocks

    def set_matrix(self, n_block_rows, rows, cols, blocks):
        U = len(rows)
        if _is_device(rows):
            self._check(self._L.adipc_gpu_set_matrix_device(self.h, n_block_rows, U, ptr(rows), ptr(cols), ptr(blocks)))
        else:
            r = np.ascontiguousarray(rows, np.uint32)
            c = np.ascontiguousarray(cols, np.uint32)
            b = np.ascontiguousarray(blocks, np.float64).reshape(-1, 9)
            self._check(self._L.adipc_gpu_set_matrix(self.h, n_block_rows, U, ptr(r), ptr(c), ptr(b)))

    def sort_stream(self, keys, vals):
        k = np.array(keys, np.uint64)
        v = np.array(vals, np.float64).reshape(-1, 9).copy()
        self._check(self._L.adipc_gpu_sort_stream(self.h, ptr(k), ptr(v), len(k)))
        return k, v

    def segment_reduce(self, O, V, n_segments, deterministic=True):
        O = np.ascontiguousarray(O, np.int32)
        V = np.ascontiguousarray(V, np.float64)
        width = 1 if V.ndim == 1 else V.shape[1]
        R = np.empty((max(n_segments, 0), width), np.float64)
        self._check(self._L.adipc_gpu_segment_reduce(self.h, ptr(O), len(O), ptr(V), V.shape[0], width, n_segments,
                                                     int(deterministic), ptr(R)))
        return R[:, 0].copy() if width == 1 else R

    def two_level_abd_reduce(self, keys, vals, n_fem, n_bodies, abd_node_body, jac36):
        k = np.ascontiguousarray(keys, np.uint64)
        v = np.ascontiguousarray(vals, np.float64).reshape(-1, 9)
        body = np.ascontiguousarray(abd_node_body, np.int32)
        jac = np.ascontiguousarray(jac36, np.float64).reshape(-1, 36)
        cap = 16 * len(k)
        ok = np.empty(cap, np.uint64)
        ov = np.empty((cap, 9), np.float64)
        n = C.c_int64()
        self._check(self._L.adipc_gpu_two_level_abd_reduce(self.h, ptr(k), ptr(v), len(k), n_fem, n_bodies, len(body),
                                                           ptr(body), ptr(jac), ptr(ok), ptr(ov), cap, C.byref(n)))
        return ok[: n.value].copy(), ov[: n.value].copy()

    def filter_pinned(self, keys, vals, pinned):
        k = np.ascontiguousarray(keys, np.uint64)
        v = np.ascontiguousarray(vals, np.float64).reshape(-1, 9)
        p = np.ascontiguousarray(pinned, np.uint8)
        ok = np.empty(len(k) + len(p), np.uint64)
        ov = np.empty((len(k) + len(p), 9), np.float64)
        n = C.c_int64()
        self._check(self._L.adipc_gpu_filter_pinned(self.h, ptr(k), ptr(v), len(k), ptr(p), len(p), ptr(ok), ptr(ov),
                                                    C.byref(n)))
        return ok[: n.value].copy(), ov[: n.value].copy()

    # -- vector arguments -----------------------------------------------------------------
    def _vec(self, a, name):
        """The C entry points read / write exactly 3 * n_block_rows doubles
        through the raw pointers: check length, dtype and layout here."""
        n, _ = self.matrix_info()
        if a is None:
            raise InvalidArgument(f"{name}: missing vector")
        if _is_device(a):
            import torch

            if a.dtype != torch.float64 or not a.is_contiguous() or a.numel() != 3 * n:
                raise InvalidArgument(f"{name}: expected a contiguous float64 tensor of {3 * n} elements")
            return a
        a = np.ascontiguousarray(a, np.float64).reshape(-1)
        if a.size != 3 * n:
            raise InvalidArgument(f"{name}: length {a.size} != 3 * n_block_rows = {3 * n}")
        return a

    # -- spmv ----------------------------------------------------------------------------
    def spmv(self, x, y=None):
        x = self._vec(x, "x")
        if _is_device(x):
            y = self._vec(y, "y")
            self._check(self._L.adipc_gpu_spmv_device(self.h, ptr(x), ptr(y)))
            return y
        y = np.empty_like(x)
        self._check(self._L.adipc_gpu_spmv(self.h, ptr(x), ptr(y)))
        return y

    # -- preconditioner ----------------------------------------------------------------------
    def set_level0_partition(self, part_of, n_parts, capacity, max_levels=4):
        p = np.ascontiguousarray(part_of, np.int32)
        self._check(self._L.adipc_gpu_set_level0_partition(self.h, ptr(p), len(p), n_parts, capacity, max_levels))

    def build_preconditioner(self, kind=_lib.PRECOND_MAS):
        self._check(self._L.adipc_gpu_build_preconditioner(self.h, kind))

    def build_mas(self, hierarchy):
        self._check(self._L.adipc_gpu_build_mas(self.h, hierarchy.h))

    def precond_levels(self):
        out = []
        for l in range(self._L.adipc_gpu_precond_n_levels(self.h)):
            nn, npart = C.c_int32(), C.c_int32()
            self._check(self._L.adipc_gpu_precond_level(self.h, l, C.byref(nn), C.byref(npart), None, None))
            n, _ = self.matrix_info()
            part = np.empty(nn.value, np.int32)
            agg = np.empty(n, np.int32)
            self._check(self._L.adipc_gpu_precond_level(self.h, l, C.byref(nn), C.byref(npart), ptr(part), ptr(agg)))
            out.append(dict(n_nodes=nn.value, n_parts=npart.value, part_of=part, agg=agg))
        return out

    def subdomain_inverse(self, level, sub):
        d = C.c_int32()
        self._check(self._L.adipc_gpu_precond_subdomain_inverse(self.h, level, sub, C.byref(d), None))
        out = np.empty(d.value * d.value, np.float64)
        self._check(self._L.adipc_gpu_precond_subdomain_inverse(self.h, level, sub, C.byref(d), ptr(out)))
        return out.reshape(d.value, d.value).T.copy()

    def shifts(self):
        s = C.c_int64()
        self._check(self._L.adipc_gpu_precond_shifts(self.h, C.byref(s)))
        return s.value

    def precond_apply(self, r, z=None):
        r = self._vec(r, "r")
        if _is_device(r):
            z = self._vec(z, "z")
            self._check(self._L.adipc_gpu_precond_apply_device(self.h, ptr(r), ptr(z)))
            return z
        z = np.empty_like(r)
        self._check(self._L.adipc_gpu_precond_apply(self.h, ptr(r), ptr(z)))
        return z

    # -- pcg ----------------------------------------------------------------------------------
    def pcg(self, b, rel_tol=1e-4, restart=250, max_iters=100000, x=None):
        it, rr, cv = C.c_int(), C.c_double(), C.c_int()
        b = self._vec(b, "b")
        if _is_device(b):
            x = self._vec(x, "x")
            self._check(self._L.adipc_gpu_pcg_device(self.h, ptr(b), rel_tol, restart, max_iters, ptr(x),
                                                     C.byref(it), C.byref(rr), C.byref(cv)))
        else:
            x = np.empty_like(b)
            self._check(self._L.adipc_gpu_pcg(self.h, ptr(b), rel_tol, restart, max_iters, ptr(x), C.byref(it),
                                              C.byref(rr), C.byref(cv)))
        return x, PcgResult(it.value, rr.value, bool(cv.value))


_default = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]
