"""The caller of the action: a conjugate-gradient loop that applies y = A x on the device
every iteration with the instance kept resident, no host round trip per action (inputs written in place
through femgpu_device_input, output written by femgpu_action_device on the same CUDA stream as the
vector updates).  The only host synchronisation is the residual-norm check every `check_every`
iterations.

The reference has no solver; this is the consumer its action exists for.  CG needs a symmetric operator:
`symmetric_problem` builds benchmark meshes whose test tabulations are the trial ones transposed
(Psi_k = Phi_k^T), which makes the mass / Laplace / Helmholtz forms of the reference map language
symmetric positive (semi-)definite.
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, List, Optional, Tuple

import numpy as np

from ._native import lib
from .action import GpuInstance, TilingParams, _call
from .form import ProblemInstance
from .mesh import mesh_problem


def symmetric_problem(form: str, dim: int, degree: int, quad_points: int, n: int, seed: int = 7) -> ProblemInstance:
    """mesh_problem with Psi_k = Phi_k^T (test space = trial space 0, same terms): a symmetric operator."""
    p = mesh_problem(form, dim, degree, quad_points, n, seed=seed)
    sig, tab = p.signature, p.tabulations
    if sig.vector_spaces or len(sig.scalar_spaces) != 1:
        raise ValueError("symmetric_problem: one scalar trial space required")
    phi = tab.scalar_phi[0]  # [terms][Q][n]
    if phi.shape[0] != sig.test_deriv_terms or phi.shape[2] != sig.test_dofs:
        raise ValueError("symmetric_problem: test space must equal the trial space")
    if not np.array_equal(p.connectivity.test_map.indices, p.connectivity.scalar_maps[0].indices):
        raise ValueError("symmetric_problem: test map must equal the trial map")
    tab.psi = np.ascontiguousarray(np.transpose(phi, (0, 2, 1)))
    p.validate()
    return p


class _CudaArray:
    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


class DeviceOperator:
    """y = A x on the device through a resident GpuInstance (scalar trial space 0 -> test space)."""

    def __init__(self, inst: GpuInstance, params: Optional[TilingParams] = None):
        import torch
        self.inst, self.params = inst, params
        p = inst.problem
        if p.signature.vector_spaces or len(p.signature.scalar_spaces) != 1:
            raise ValueError("DeviceOperator: one scalar trial space required")
        self.n = int(p.output_size)
        if p.connectivity.scalar_maps[0].global_count != self.n:
            raise ValueError("DeviceOperator: square operators only (trial and test sizes differ)")
        xp = C.c_void_p()
        _call(lib().femgpu_device_input(inst.handle, 0, C.byref(xp)))
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.x = torch.as_tensor(_CudaArray(xp.value, self.n), device=self.dev)  # the instance's input buffer
        self.launches = 0

    def apply(self, v, out) -> None:
        """out = A v (both float64 device tensors); ordered on torch's current stream."""
        import torch
        self.x.copy_(v)
        stream = torch.cuda.current_stream(self.dev).cuda_stream or 1  # 0 = legacy default stream -> cudaStreamLegacy
        self.inst.action_device(self.params, y_dev=out.data_ptr(), stream=stream)
        self.launches += 1


def cg(apply: Callable, b, x0=None, rtol: float = 1e-10, maxiter: int = 1000,
       check_every: int = 1, dot: Optional[Callable] = None) -> Tuple[object, int, List[float]]:
    """Conjugate gradients for A x = b with A symmetric positive definite on span(b).
    `apply(v, out)` writes A v into out; vectors are torch tensors (any device); `dot` defaults to
    torch.dot (a distributed caller passes an all-reduced dot).  Returns (x, iterations, residual norms)."""
    import torch
    dot = dot or (lambda a, c: torch.dot(a, c))
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    r = b.clone()
    if x0 is not None:
        ax = torch.empty_like(b)
        apply(x, ax)
        r -= ax
    p = r.clone()
    ap = torch.empty_like(b)
    rr = dot(r, r)
    bnorm = float(torch.sqrt(dot(b, b)))
    hist = [float(torch.sqrt(rr))]
    if hist[0] <= rtol * bnorm:
        return x, 0, hist
    for it in range(1, maxiter + 1):
        apply(p, ap)
        alpha = rr / dot(p, ap)
        x.add_(alpha * p)
        r.sub_(alpha * ap)
        rr_new = dot(r, r)
        p.mul_(rr_new / rr).add_(r)
        rr = rr_new
        if it % check_every == 0:
            hist.append(float(torch.sqrt(rr)))
            if hist[-1] <= rtol * bnorm:
                return x, it, hist
    return x, maxiter, hist


def native_cg(inst: GpuInstance, b, x0=None, rtol: float = 1e-10, maxiter: int = 1000, check_every: int = 10,
              params: Optional[TilingParams] = None):
    """CG inside libfemgpu (femgpu_cg, csrc/cg.cu): the whole loop on the instance stream, fused update
    kernels, deterministic reductions.  b, x0: float64 CUDA tensors.  Returns (x, iterations, relative
    residual)."""
    import torch
    from .action import _sched
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    torch.cuda.synchronize()  # b and x are ready before the instance stream reads them
    it = C.c_int32()
    rel = C.c_double()
    sp = _sched(params)
    _call(lib().femgpu_cg(inst.handle, sp[0] if sp else None, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()),
                          rtol, maxiter, check_every, C.byref(it), C.byref(rel)))
    return x, it.value, rel.value


def dist_cg(plan_, dist_apply: Callable, b_local, rtol: float = 1e-10, maxiter: int = 1000, check_every: int = 1):
    """Distributed CG over the cell partition of dist.build_plan (one rank per GPU).

    Vectors live in the rank's local test numbering (owned rows + ghosts; the trial space is numbered
    like the test space).  `dist_apply(v, out)` is the complete distributed action -- ghost inputs
    pulled from their owners, local action, partial rows pushed to their owners -- either on the
    device (DistOperator: csrc/halo.cu, GPU to GPU) or emulated on the host (dist.host_halo_action);
    afterwards only owned rows are meaningful and ghost rows are zeroed.  Dots run over owned rows and
    are all-reduced; each all-reduce also orders the ranks' input updates after every rank's pulls."""
    import torch
    import torch.distributed as dist
    owned = torch.as_tensor(plan_.owned_mask, device=b_local.device)

    def dot(a, c):
        t = torch.sum(a[owned] * c[owned]).reshape(1).cpu()
        dist.all_reduce(t)
        return t[0].to(a.device)

    def apply(v, out):
        dist_apply(v, out)
        out[~owned] = 0.0

    return cg(apply, b_local, rtol=rtol, maxiter=maxiter, check_every=check_every, dot=dot)


class DistOperator:
    """Distributed y = A x on the devices: a dist.DistInstance (scalar trial space 0 numbered like the
    test space); apply(v, out) writes v into the instance input, runs the halo action into out."""

    def __init__(self, di):
        import torch
        self.di = di
        p = di.plan.local
        if p.signature.vector_spaces or len(p.signature.scalar_spaces) != 1:
            raise ValueError("DistOperator: one scalar trial space required")
        n = int(p.output_size)
        xp = C.c_void_p()
        _call(lib().femgpu_device_input(di.inst.handle, 0, C.byref(xp)))
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.x = torch.as_tensor(_CudaArray(xp.value, n), device=self.dev)
        self.launches = 0

    def apply(self, v, out) -> None:
        """Ordered on torch's current stream.  Ranks sharing a device in one process must each run on
        their own stream (torch.cuda.ExternalStream(inst.stream())), never the legacy default stream."""
        import torch
        self.x.copy_(v)
        stream = torch.cuda.current_stream(self.dev).cuda_stream or 1
        self.di.action(y_dev=out.data_ptr(), stream=stream)
        self.launches += 1
