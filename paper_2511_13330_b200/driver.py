"""Host-side driver: device buffers, sub-batching and multi-GPU partitioning around
the C ABI (B3 in SURVEY.md).  Plumbing only -- every arithmetic step of the hot path
runs inside libqal.so.

* PulseBatch  -- configs[2]-style batches: per-pulse drift, shared controls basis;
                 the batch is processed in sub-batches whose gradient workspace fits
                 HBM; across ranks the pulses are partitioned (no data-path collective).
* time_shard_propagator -- configs[3]-style long horizons: rank r owns the slice range
                 [r N/G, (r+1) N/G), folds it into one partial (same chunk/tree shape
                 for every G), all-gathers the G partials and combines them in order
                 (later rank on the LEFT, Eq. 15).
"""
from __future__ import annotations

import ctypes
import math

import torch

from . import qal

C128 = torch.complex128
F64 = torch.float64


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class PulseBatch:
    """Forward + gradient for a batch of pulses with per-pulse drift Hamiltonians.

    Inputs are device tensors: H0 [B][d][d], Hc [J][d][d], C [K][d][d], u [B][N][J], V [d][d].
    ``step()`` runs the whole hot path (a2 Liouvillian, a3-a5 propagator, a6 fidelity,
    a7 gradient) and leaves F [B] and grad [B][N][J] in preallocated device buffers.
    """

    def __init__(self, H0, Hc, C, u, V, T, *, sub_batch=None, want_grad=True, magnus_order=4, stream=None,
                 structure="dense"):
        self.H0, self.Hc, self.C, self.u, self.V = H0, Hc, C, u, V
        self.B, self.N, self.J = u.shape[0], u.shape[1], Hc.shape[0]
        self.d = V.shape[0]
        self.n = self.d * self.d
        self.T = float(T)
        self.order = magnus_order
        self.want_grad = want_grad
        if structure not in ("dense", "blocks"):
            raise ValueError(f"structure must be 'dense' or 'blocks', got {structure!r}")
        self.structure = structure
        dev = u.device
        self.stream = stream
        self.L0 = torch.empty((self.B, self.n, self.n), dtype=C128, device=dev)
        self.Lc = torch.empty((self.J, self.n, self.n), dtype=C128, device=dev)
        self.F = torch.empty(self.B, dtype=F64, device=dev)
        self.grad = torch.empty_like(u) if want_grad else None
        self.status = torch.zeros(self.B, dtype=torch.int32, device=dev)
        op = qal.QAL_OP_FIDELITY_GRAD if want_grad else qal.QAL_OP_FIDELITY
        self.launches = 0
        if structure == "dense":
            self.sub = self.B if sub_batch is None else min(sub_batch, self.B)
            self.ws_bytes = qal.workspace_bytes(op, self.n, self.sub, self.N, self.J, 0)
        else:
            # coherence-block path: the plan is detected once from the generator
            # basis of pulse 0; every step re-verifies every pulse on the device and reports a pulse whose
            # L0_b (or the shared L_j) couples two blocks as QAL_ERR_STRUCTURE in status[b]
            self._build_basis()
            self.plan = qal.qal_block_plan_build(torch.cat([self.L0[:1], self.Lc]), mirror=True)
            self.L0p = torch.empty((self.B, self.plan.packed), dtype=C128, device=dev)
            self.Lcp = torch.empty((self.J, self.plan.packed), dtype=C128, device=dev)
            if sub_batch is None:
                # image workspace (3 packed images per slice) within ~80 GB of HBM (at most 45% of the
                # device, so a dense reference run fits beside it), rounded to whole multiples of
                # 2 x SMs pulses.  Larger sub-batches keep more pulse chains in flight in the fused
                # forward (one CTA slot per pulse): configs[2] 888 -> 1776 pulses per launch took the
                # forward from 88.6 to 79.3 ms per step (round 1).  Batches below 8 x SMs pulses run the
                # split forward instead (qal_api.cu blk_split_forward)
                props = torch.cuda.get_device_properties(dev)
                per = 3 * self.N * self.plan.packed * 16
                wave = 2 * props.multi_processor_count
                sub_batch = int(min(80e9, 0.45 * props.total_memory) // per)
                if sub_batch >= wave:
                    sub_batch -= sub_batch % wave
                sub_batch = max(1, min(self.B, sub_batch))
            self.sub = min(sub_batch, self.B)
            self.ws_bytes = qal.block_workspace_bytes(self.plan, op, self.sub, self.N)
        self.ws = torch.empty(max(self.ws_bytes, 1), dtype=torch.uint8, device=dev)
        self._pipe = None

    def _s(self):
        s = torch.cuda.current_stream() if self.stream is None else self.stream
        return ctypes.c_void_p(s.cuda_stream)

    def _build_basis(self):
        lib = qal.load()
        nc = 0 if self.C is None else self.C.shape[0]
        rc = lib.qal_build_liouvillian(self.d, self.B, _p(self.H0), self.J, _p(self.Hc), nc, _p(self.C), 0,
                                       _p(self.L0), _p(self.Lc), None, self._s())
        qal._check(rc, "qal_build_liouvillian")
        return lib.qal_last_launch_count()

    def subs(self):
        """The sub-batches (first pulse, pulses) one step runs, in order."""
        return [(b0, min(self.sub, self.B - b0)) for b0 in range(0, self.B, self.sub)]

    def step(self, hooks=None):
        """One step on the device-resident inputs.  `hooks` (step_host's copy pipeline): an object with
        after_basis(), before_sub(i, b0, nb) and after_sub(i, b0, nb), called as the work is enqueued."""
        lib = qal.load()
        st = self._s()
        if hooks is not None:
            hooks.before_basis()
        launches = self._build_basis()
        if hooks is not None:
            hooks.after_basis()
        if self.structure == "blocks":
            return self._step_blocks(lib, st, launches, hooks)
        plane = self.n * self.n
        for i, (b0, nb) in enumerate(self.subs()):
            if hooks is not None:
                hooks.before_sub(i, b0, nb)
            rc = lib.qal_fidelity_grad(
                self.d, nb, self.N, self.T, self.order, qal.QAL_CTRL_PWC, self.J,
                ctypes.c_void_p(self.u.data_ptr() + b0 * self.N * self.J * 8),
                ctypes.c_void_p(self.L0.data_ptr() + b0 * plane * 16), plane, _p(self.Lc), None, 0, _p(self.V),
                ctypes.c_void_p(self.F.data_ptr() + b0 * 8),
                ctypes.c_void_p(self.grad.data_ptr() + b0 * self.N * self.J * 8) if self.want_grad else None,
                None, ctypes.c_void_p(self.status.data_ptr() + b0 * 4), _p(self.ws), self.ws_bytes, st)
            qal._check(rc, "qal_fidelity_grad")
            launches += lib.qal_last_launch_count()
            if hooks is not None:
                hooks.after_sub(i, b0, nb)
        self.launches = launches
        return self.F, self.grad

    def _step_blocks(self, lib, st, launches, hooks=None):
        pl = ctypes.byref(self.plan)
        for src, dst in ((self.L0, self.L0p), (self.Lc, self.Lcp)):
            qal._check(lib.qal_block_pack(pl, src.shape[0], _p(src), _p(dst), None, st), "qal_block_pack")
            launches += lib.qal_last_launch_count()
        P = self.plan.packed
        for i, (b0, nb) in enumerate(self.subs()):
            if hooks is not None:
                hooks.before_sub(i, b0, nb)
            rc = lib.qal_block_fidelity_grad(
                pl, nb, self.N, self.T, self.order, qal.QAL_CTRL_PWC, self.J,
                ctypes.c_void_p(self.u.data_ptr() + b0 * self.N * self.J * 8),
                ctypes.c_void_p(self.L0p.data_ptr() + b0 * P * 16), P, _p(self.Lcp), None, 0, _p(self.V),
                ctypes.c_void_p(self.F.data_ptr() + b0 * 8),
                ctypes.c_void_p(self.grad.data_ptr() + b0 * self.N * self.J * 8) if self.want_grad else None,
                None, ctypes.c_void_p(self.status.data_ptr() + b0 * 4), _p(self.ws), self.ws_bytes, st)
            qal._check(rc, "qal_block_fidelity_grad")
            launches += lib.qal_last_launch_count()
            if hooks is not None:
                hooks.after_sub(i, b0, nb)
        # the structure check of this step's operators, per pulse (after the calls above, which reset
        # their status slices on entry): L0_b -> status[b]; a shared L_j -> every pulse
        qal._check(lib.qal_block_check(pl, self.B, _p(self.L0), 0, _p(self.status), self.B, st), "qal_block_check")
        if self.J > 0:
            qal._check(lib.qal_block_check(pl, self.J, _p(self.Lc), 1, _p(self.status), self.B, st),
                       "qal_block_check")
        launches += 1 + (self.J > 0)
        self.launches = launches
        return self.F, self.grad

    def step_host(self, hH0, hu, hF, hg):
        """One step from pinned host inputs to pinned host results (the end-to-end call): H0 [B][d][d]
        and u [B][N][J] are copied in, F [B] and grad [B][N][J] copied out, all on two copy streams that
        overlap the compute: sub-batch i's controls go in as soon as the previous step's sub-batch i is done
        with them (so step s + 1's inputs stream in under step s), its results go out as soon as it is done
        (under sub-batch i + 1).  The next step's compute is not held back by this step's last copy-out;
        `host_fence()` orders the caller's stream after it (an event recorded there afterwards marks the
        results in host memory) and `synchronize_host()` waits for it on the host."""
        if self._pipe is None:
            self._pipe = _CopyPipeline(self)
        return self._pipe.run(hH0, hu, hF, hg)

    def host_fence(self):
        """Order the caller's stream after the last step_host's copy-out."""
        if self._pipe is not None:
            self._pipe.fence()

    def synchronize_host(self):
        """Wait until the last step_host's results are in host memory."""
        self.host_fence()
        (torch.cuda.current_stream() if self.stream is None else self.stream).synchronize()

    def structure_ok(self) -> bool:
        """False if the last step's device check found an operator coupling two blocks of the plan
        (those pulses carry QAL_ERR_STRUCTURE in `status`; synchronises)."""
        return self.structure == "dense" or not bool((self.status == qal.QAL_ERR_STRUCTURE).any())


class _CopyPipeline:
    """PulseBatch.step_host's copy streams and the events that order them against the compute stream
    (across steps: a buffer is overwritten only after its previous reader is done)."""

    def __init__(self, eng):
        self.eng = eng
        dev = eng.u.device
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        n = len(eng.subs())
        ev = lambda: torch.cuda.Event()  # noqa: E731
        self.h0_in, self.h0_free = ev(), ev()              # H0 copied in / basis build done with it
        self.u_in = [ev() for _ in range(n)]               # sub-batch i's controls copied in
        self.u_free = [ev() for _ in range(n)]             # sub-batch i's compute done (u read, F / grad written)
        self.out_done = [ev() for _ in range(n)]           # sub-batch i's results copied out
        self.started = False

    def run(self, hH0, hu, hF, hg):
        eng = self.eng
        comp = torch.cuda.current_stream() if eng.stream is None else eng.stream
        first = not self.started
        self.started = True
        subs = eng.subs()
        with torch.cuda.stream(self.h2d):
            if not first:
                self.h2d.wait_event(self.h0_free)
            eng.H0.copy_(hH0, non_blocking=True)
            self.h0_in.record(self.h2d)
            for i, (b0, nb) in enumerate(subs):
                if not first:
                    self.h2d.wait_event(self.u_free[i])
                eng.u[b0:b0 + nb].copy_(hu[b0:b0 + nb], non_blocking=True)
                self.u_in[i].record(self.h2d)
        pipe = self

        class Hooks:
            def before_basis(self):
                comp.wait_event(pipe.h0_in)

            def after_basis(self):
                pipe.h0_free.record(comp)

            def before_sub(self, i, b0, nb):
                comp.wait_event(pipe.u_in[i])
                if not first:
                    comp.wait_event(pipe.out_done[i])      # F / grad of sub-batch i copied out last step

            def after_sub(self, i, b0, nb):
                pipe.u_free[i].record(comp)
                with torch.cuda.stream(pipe.d2h):
                    pipe.d2h.wait_event(pipe.u_free[i])
                    hF[b0:b0 + nb].copy_(eng.F[b0:b0 + nb], non_blocking=True)
                    if eng.grad is not None and hg is not None:
                        hg[b0:b0 + nb].copy_(eng.grad[b0:b0 + nb], non_blocking=True)
                    pipe.out_done[i].record(pipe.d2h)

        eng.step(hooks=Hooks())
        return hF, hg

    def fence(self):
        comp = torch.cuda.current_stream() if self.eng.stream is None else self.eng.stream
        comp.wait_event(self.out_done[len(self.eng.subs()) - 1])


def shard_range(total: int, world: int, rank: int):
    """Contiguous equal shard [lo, hi) of `total` units for `rank` (total % world == 0)."""
    if total % world:
        raise ValueError(f"{total} units do not split over {world} ranks")
    per = total // world
    return rank * per, (rank + 1) * per


def time_shard_chunk(n_slices: int, world_max: int = 8) -> int:
    """Chunk size keyed to N only (A16): every rank's range is a union of whole subtrees
    for any G <= world_max dividing N, so the product is bit-identical across G."""
    base = n_slices
    for g in (world_max, 4, 2, 1):
        if n_slices % g == 0:
            base = n_slices // g
            break
    c = 1
    while c < 64 and base % (2 * c) == 0:
        c *= 2
    return c


def gather_partials(Q, group=None):
    """All-gather every rank's partial product [n][n] -> [G][n][n] in rank order (NCCL over
    NVLink on GPUs, gloo on CPU).  Complex tensors travel as their real view."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return Q.unsqueeze(0)
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(Q.shape), dtype=Q.dtype, device=Q.device)
    dist.all_gather_into_tensor(torch.view_as_real(out).reshape(-1), torch.view_as_real(Q.contiguous()).reshape(-1),
                                group=group)
    return out


def gather_results(F, grad=None, group=None):
    """configs[2] / configs[4] result exchange: every rank's F [B_r] (and grad
    [B_r][N][J]) -> the whole batch [G B_r] (...) in rank order, i.e. in global pulse order when rank r
    owns pulses [r B_r, (r+1) B_r) -- all_gather_into_tensor (NCCL over NVLink on GPUs, gloo on CPU).
    With no process group (one rank) the local tensors are returned as they are."""
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return F, grad
    world = dist.get_world_size(group)
    Fa = torch.empty((world * F.shape[0],), dtype=F.dtype, device=F.device)
    dist.all_gather_into_tensor(Fa, F.contiguous(), group=group)
    ga = None
    if grad is not None:
        ga = torch.empty((world * grad.shape[0],) + tuple(grad.shape[1:]), dtype=grad.dtype, device=grad.device)
        dist.all_gather_into_tensor(ga.reshape(-1), grad.contiguous().reshape(-1), group=group)
    return Fa, ga


def ordered_combine(parts, product=None, stream=None, plan=None):
    """Lambda = Q_{G-1} ... Q_0 (Eq. 15, later rank on the LEFT) from the gathered partials [G][n][n]
    (or [G][packed] with a block plan), with the same balanced-tree shape as qal_ordered_product.
    `product(list_or_tensor)` may be swapped for tests; the default is the library's tree kernel."""
    if product is not None:
        return product(parts)
    if plan is not None:
        return qal.qal_block_ordered_product(plan, parts.unsqueeze(0).contiguous(), stream=stream)[0]
    return qal.qal_ordered_product(parts.unsqueeze(0).contiguous(), stream=stream)[0]


def local_partial(L0, Lc, Lcomm, u_local, T, n_slices, k0, *, ctrl_mode, magnus_order=4, stream=None, plan=None):
    """This rank's partial Q = U_{k0+count-1} ... U_{k0}: chunk fold (chunk keyed to N only) + tree.
    With a block plan the basis is packed (qal_block_pack) and Q is a packed matrix."""
    count = u_local.shape[1]
    chunk = time_shard_chunk(n_slices)
    if count % chunk:
        raise ValueError(f"slice range {count} is not a multiple of the chunk {chunk}")
    if plan is not None:
        parts = qal.qal_block_expm_slices(plan, L0, Lc, u_local, T, n_slices, k0=k0, count=count,
                                          magnus_order=magnus_order, ctrl_mode=ctrl_mode, Lcommp=Lcomm,
                                          chunk=chunk, stream=stream)
        return qal.qal_block_ordered_product(plan, parts, stream=stream)[0]
    _, parts = qal.qal_magnus_expm_slices(L0, Lc, u_local, T, n_slices, k0=k0, count=count,
                                          magnus_order=magnus_order, ctrl_mode=ctrl_mode, Lcomm=Lcomm,
                                          chunk=chunk, stream=stream)
    return qal.qal_ordered_product(parts, stream=stream)[0]


def time_shard_propagator(L0, Lc, Lcomm, u_local, T, n_slices, k0, *, ctrl_mode, magnus_order=4, group=None,
                          stream=None, plan=None):
    """configs[3]: this rank's slices [k0, k0 + count) -> local partial -> all-gather -> ordered
    combine.  Returns Lambda (identical on every rank; packed when a block plan is given, so the
    all-gather moves 14 KB per rank instead of 64 KB)."""
    Q = local_partial(L0, Lc, Lcomm, u_local, T, n_slices, k0, ctrl_mode=ctrl_mode, magnus_order=magnus_order,
                      stream=stream, plan=plan)
    return ordered_combine(gather_partials(Q, group), stream=stream, plan=plan)


def calibrate(H0, Hc, C, u0, T, Pproj, G, *, iters=200, lr=1e-2, beta1=0.9, beta2=0.999, eps=1e-8,
              magnus_order=4, stream=None, structure="dense"):
    """NEXT f1 -- the paper's calibration loop: Adam over the PWC coefficient matrix
    u [B][M][J] minimising the Eq. 16-17 loss 1/4 ||P^dag Lambda P - G||_F^2, every step on the
    device: forward (qal_propagator_forward) -> loss + cotangent (qal_logical_loss) -> gradient
    (qal_propagator_vjp, one adjoint Frechet derivative per slice; the paper's autodiff hit a
    memory wall here) -> qal_adam_step.  Returns dict(u, loss_history [iters, B],
    best_u, best_loss); no host synchronisation inside the loop.

    structure="blocks": the coherence-block path.  The Eq. 16-17 cotangent
    C = 1/2 P (Pi - G)^dag P^dag preserves Hermiticity when G is real (Pi = P^dag Lambda P is real for a
    Hermiticity-preserving Lambda and the Hermitian DFS projectors), so it packs exactly; the forward of
    each step is recomputed inside qal_block_propagator_vjp (the block path has no split forward/vjp)."""
    u = u0.clone().contiguous()
    L0, Lc, _ = qal.qal_build_liouvillian(H0, Hc, C, stream=stream)
    m = torch.zeros_like(u)
    v = torch.zeros_like(u)
    hist = torch.empty((iters, u.shape[0]), dtype=F64, device=u.device)
    best = torch.full((u.shape[0],), float("inf"), dtype=F64, device=u.device)
    best_u = u.clone()
    N = u.shape[1]
    if structure == "blocks":
        if G.is_complex() and bool((G.imag != 0).any()):
            raise ValueError("the block path needs a real logical target G (Hermiticity-preserving cotangent)")
        plan = qal.qal_block_plan_build(torch.cat([L0, Lc]), mirror=True)
        L0p, _ = qal.qal_block_pack(plan, L0, check=False, stream=stream)
        Lcp, _ = qal.qal_block_pack(plan, Lc, check=False, stream=stream)
        ch = N
        for t in range(1, iters + 1):
            parts = qal.qal_block_expm_slices(plan, L0p, Lcp, u, T, N, chunk=ch, magnus_order=magnus_order,
                                              stream=stream)
            Lam = qal.qal_block_unpack(plan, parts[:, 0], stream=stream)
            loss, cot = qal.qal_logical_loss(Lam, Pproj, G, stream=stream)
            hist[t - 1] = loss
            better = loss < best
            best = torch.where(better, loss, best)
            best_u[better] = u[better]
            cotp, _ = qal.qal_block_pack(plan, cot, check=False, stream=stream)
            g, _ = qal.qal_block_propagator_vjp(plan, L0p, Lcp, u, T, N, cotp, magnus_order=magnus_order,
                                                stream=stream)
            qal.qal_adam_step(u, g, m, v, t, lr, beta1, beta2, eps, stream=stream)
        return {"u": u, "loss_history": hist, "best_u": best_u, "best_loss": best}
    sess = qal.GradientSession(L0, Lc, u, T, N, magnus_order=magnus_order, stream=stream)
    for t in range(1, iters + 1):
        Lam = sess.forward()
        loss, cot = qal.qal_logical_loss(Lam, Pproj, G, stream=stream)
        hist[t - 1] = loss
        better = loss < best
        best = torch.where(better, loss, best)
        best_u[better] = u[better]
        g = sess.vjp(cot)
        qal.qal_adam_step(u, g, m, v, t, lr, beta1, beta2, eps, stream=stream)
    return {"u": u, "loss_history": hist, "best_u": best_u, "best_loss": best}


def segment_seeds(Qs, C, product):
    """Seed algebra of the time-sharded gradient (NEXT f2).  Qs: the time-ordered partial products
    Q_0 .. Q_{S-1} of consecutive slice segments (over all ranks), C: the cotangent of the objective
    at Lambda = Q_{S-1} ... Q_0.  For segment s with local prefixes P_k^loc (P_init = I),
        G_k = P_k^loc X'_{k+1},   X'_{end of s} = (Q_{s-1} ... Q_0) C (Q_{S-1} ... Q_{s+1})
    so the vjp of every segment runs on its own slices with the seed X'_s (no recomputation).
    `product(list)` = ordered product of a time-ordered list (later on the LEFT).
    Returns the list of seeds."""
    S = len(Qs)
    seeds = []
    for s in range(S):
        prefix = product(Qs[:s]) if s > 0 else None
        suffix = product(Qs[s + 1:]) if s + 1 < S else None
        chain = [x for x in (suffix, C, prefix) if x is not None]   # prefix C suffix  (time order reversed)
        seeds.append(product(chain) if len(chain) > 1 else chain[0])
    return seeds


def rank_seed(ranks, C, rank, combine, matmul):
    """Cotangent of rank `rank`'s own partial Q_r in a time-sharded objective (NEXT f2): with
    Lambda = Q_{G-1} ... Q_0 (later rank on the LEFT, Eq. 15) and dL = Re Tr(C dLambda),
        dL = Re Tr(C A_r dQ_r B_r) = Re Tr((B_r C A_r) dQ_r),
    B_r = Q_{r-1} ... Q_0 (earlier ranks), A_r = Q_{G-1} ... Q_{r+1} (later ranks); so the seed is
    B_r C A_r.  ranks: the gathered partials [G][...]; combine(parts) = their ordered product;
    matmul(X, Y) = X Y (dense or packed).  Identity factors are skipped (rank 0 / rank G-1)."""
    G = ranks.shape[0]
    if rank > 0:                     # earlier ranks sit right of the local prefix: C <- B_r C
        C = matmul(combine(ranks[:rank]), C)
    if rank + 1 < G:                 # later ranks sit left of the local suffix: C <- C A_r
        C = matmul(C, combine(ranks[rank + 1:]))
    return C


def time_sharded_gradient(L0, Lc, Lcomm, u_local, T, n_slices, k0, *, ctrl_mode, cotangent, magnus_order=4,
                          sub=64, group_subsegments=2048, group=None, stream=None, plan=None):
    """NEXT f2 -- gradient of an objective over a long horizon, time-sharded over the ranks, with
    log-depth parallelism inside each rank.  Rank r owns slices [k0, k0 + count) of ONE pulse
    (u_local [1][count][...]):
      1. sub-segment partials Q_s (s < S = count/sub): chunk fold, all sub-segments in parallel;
      2. exclusive prefix / suffix products of the Q_s: Hillis-Steele scan (qal_ordered_scan);
      3. all-gather of the rank totals (NCCL); Lambda; C = cotangent(Lambda);
         rank seed C_r = (ranks before) C (ranks after)... as matrices: B_r C A_r with
         B_r = Q_{r-1}..Q_0 (earlier ranks) on the left of C and A_r = Q_{G-1}..Q_{r+1} on the right
      4. sub-segment seeds pre_s C_r suf_s (segment_seeds, batched);
      5. the VJP of all sub-segments as one batch of short "pulses" (qal_propagator_forward / _vjp),
         in groups so the stored images fit HBM.
    With a block plan (coherence-block path) the basis is packed, every matrix above is packed, the
    cotangent must return a packed Hermiticity-preserving C, and step 5 is qal_block_propagator_vjp.
    Returns (Lambda, grad of the local slices)."""
    count = u_local.shape[1]
    if count % sub:
        raise ValueError("sub must divide the rank's slice count")
    S = count // sub
    if plan is not None:
        return _time_sharded_gradient_blocks(plan, L0, Lc, Lcomm, u_local, T, n_slices, k0, ctrl_mode=ctrl_mode,
                                             cotangent=cotangent, magnus_order=magnus_order, sub=sub,
                                             group_subsegments=group_subsegments, group=group, stream=stream)
    _, parts = qal.qal_magnus_expm_slices(L0, Lc, u_local, T, n_slices, k0=k0, count=count,
                                          magnus_order=magnus_order, ctrl_mode=ctrl_mode, Lcomm=Lcomm, chunk=sub,
                                          stream=stream)
    pre, suf = qal.qal_ordered_scan(parts, stream=stream)                        # [1][S]
    Q_rank = qal.qal_batched_matmul(parts[:, S - 1], pre[:, S - 1], stream=stream)[0]
    ranks = gather_partials(Q_rank, group)                                        # [G][n][n]
    rank = _rank(group)
    Lam = ordered_combine(ranks, stream=stream)
    C = rank_seed(ranks, cotangent(Lam), rank, lambda P: ordered_combine(P, stream=stream),
                  lambda X, Y: qal.qal_batched_matmul(X.unsqueeze(0), Y.unsqueeze(0), stream=stream)[0])
    tmp = qal.qal_batched_matmul(C.unsqueeze(0), suf[0], stream=stream)          # C_r suf_s
    seeds = qal.qal_batched_matmul(pre[0], tmp, stream=stream)                    # pre_s C_r suf_s
    del tmp, pre, suf, parts
    us = u_local[0].reshape((S, sub) + tuple(u_local.shape[2:]))
    grad = torch.empty_like(us)
    for g0 in range(0, S, group_subsegments):
        g1 = min(S, g0 + group_subsegments)
        sess = qal.GradientSession(L0, Lc, us[g0:g1].contiguous(), T, n_slices, k0=0, magnus_order=magnus_order,
                                   ctrl_mode=ctrl_mode, Lcomm=Lcomm, stream=stream)
        sess.forward()
        grad[g0:g1] = sess.vjp(seeds[g0:g1].contiguous())
        del sess
    return Lam, grad.reshape(u_local.shape)


def _time_sharded_gradient_blocks(plan, L0p, Lcp, Lcommp, u_local, T, n_slices, k0, *, ctrl_mode, cotangent,
                                  magnus_order, sub, group_subsegments, group, stream):
    """Block path of time_sharded_gradient: ONE forward over all sub-segments (qal_block_propagator_forward:
    its per-sub-segment Lambda are the partials Q_s, and it keeps every U_k, P_k and (m, s) choice), then
    the scans / all-gather / seeds, then only the reverse pass on the stored forward
    (qal_block_propagator_backward) -- no slice is exponentiated twice.  The stored forward takes
    3 packed images per slice (45 GB for 2^20 slices at G = 1); group_subsegments is not used here."""
    count = u_local.shape[1]
    S = count // sub
    bmm = lambda A, B: qal.qal_block_batched_matmul(plan, A, B, stream=stream)  # noqa: E731
    us = u_local[0].reshape((S, sub) + tuple(u_local.shape[2:])).contiguous()
    sess = qal.BlockGradientSession(plan, L0p, Lcp, us, T, n_slices, magnus_order=magnus_order,
                                    ctrl_mode=ctrl_mode, Lcommp=Lcommp, stream=stream)
    parts = sess.forward().unsqueeze(0)                                               # [1][S][packed]
    pre, suf = qal.qal_block_ordered_scan(plan, parts, stream=stream)
    Q_rank = bmm(parts[0, S - 1], pre[0, S - 1])[0]
    ranks = gather_partials(Q_rank, group)                                             # [G][packed]
    rank = _rank(group)
    Lam = ordered_combine(ranks, stream=stream, plan=plan)
    C = rank_seed(ranks, cotangent(Lam), rank, lambda P: ordered_combine(P, stream=stream, plan=plan),
                  lambda X, Y: bmm(X, Y)[0])
    seeds = bmm(pre[0], bmm(C, suf[0]))                                                # pre_s C_r suf_s
    del pre, suf, parts
    grad = sess.vjp(seeds)
    del sess
    return Lam, grad.reshape(u_local.shape)


def _rank(group=None):
    import torch.distributed as dist
    return dist.get_rank(group) if (dist.is_available() and dist.is_initialized()) else 0


def fp64_peak(sink, blocks, seconds=0.2, kind=0):
    """Measured FP64 peak (K0 probe, DMMA.8x8x4 by default) in TFLOP/s on the current device."""
    iters = 2000
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    qal.qal_fp64_peak_probe(kind, blocks, iters, sink)      # warm-up
    torch.cuda.synchronize()
    start.record()
    fl = qal.qal_fp64_peak_probe(kind, blocks, iters, sink)
    end.record()
    end.synchronize()
    ms = start.elapsed_time(end)
    iters = max(1, int(iters * seconds * 1e3 / max(ms, 1e-3)))
    best = 0.0
    for _ in range(3):
        start.record()
        fl = qal.qal_fp64_peak_probe(kind, blocks, iters, sink)
        end.record()
        end.synchronize()
        best = max(best, fl / (start.elapsed_time(end) * 1e-3) / 1e12)
    return best


MATMUL_FLOPS_64 = 8.0 * 64 ** 3     # one 64x64 complex product (ZGEMM convention)


def complex_product_flops(n: int = 64) -> float:
    """Algorithmic flops of one n x n complex product as the library executes it: 2 n^3 per real
    multiplication, 3 of them for the Gauss (3M) form -> 6 n^3 (a 3M product counts
    6 n^3 so the roofline fraction is not inflated), 8 n^3 for the default 4M build."""
    return 2.0 * n ** 3 * qal.real_mults_per_complex_product()


def stage_flops(products: int, stage: str = "") -> float:
    """Algorithmic flops of a profiling-window counter: the dense stages count 64x64 complex
    products, the coherence-block stages (qal.FLOP_STAGES) count flops directly."""
    if stage in qal.FLOP_STAGES:
        return float(products)
    return products * complex_product_flops(64)


__all__ = ["PulseBatch", "shard_range", "time_shard_chunk", "time_shard_propagator", "ordered_combine",
           "gather_partials", "gather_results", "rank_seed", "local_partial", "calibrate", "segment_seeds", "time_sharded_gradient", "fp64_peak",
           "MATMUL_FLOPS_64", "complex_product_flops", "stage_flops", "math"]
