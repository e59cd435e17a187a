"""Row-block sharded QMCUR across the GPUs of one node.

Rank g of G owns rows [g m/G, (g+1) m/G) of X (generated or loaded locally; a
34 GB matrix never moves).  The path's real exchange steps, each one
torch.distributed collective on device buffers (NCCL over NVLink):

  K1  column sums     numpy's *sequential* axis-0 order continued rank to rank
                      (send/recv chain pipelined by column chunks), then broadcast;
      row sums        local (rows are whole);
      flat total      each rank's rows are one complete subtree of numpy's
                      pairwise tree (checked); G partials all-gathered and
                      combined in the tree's own order -> bit-identical to numpy;
      row normaliser  all-gather of the m row weights.
  K2  draws           identical on every rank (same weights, same PCG64 stream).
  K3  C = X[:, J]     rows local;  R = X[I, :]: owners copy their rows, all-gather,
                      one device gather by an owner-slot table (byte copies -> bit-exact).
  K4  pinv(C)         distributed CholeskyQR2: all-reduce of the c x c Grams;
      pinv(R)         R replicated -> factored redundantly.
  K6  Y_g = X_g Q_R (qcur_xq: INT8 tensor cores, in row chunks when the residues are large);
      M = sum_g Q_C,g^H Y_g (all-reduce of c x r);  U replicated.
  K9  error partials  local fused kernel; 4 statistics all-gathered and summed
                      in rank order.

The orchestration is written against two small interfaces — ``ops`` (device
computation; GpuOps calls the C ABI) and ``comm`` (collectives) — so the
multi-rank logic is exercised on CPU with gloo in tests/test_rowshard.py (with
a numpy ops object supplied by the test), and on the GPU through GpuOps.
"""
from __future__ import annotations

import math

import numpy as np

from . import _native


# ---------------------------------------------------------------------------
# the flat pairwise tree over row blocks
# ---------------------------------------------------------------------------
def subtree_aligned(total: int, world: int) -> bool:
    """True when numpy's pairwise recursion over `total` elements (split at
    n2 = n/2 - (n/2 % 8)) yields exactly `world` equal leaves at depth
    log2(world): then each rank's block is one complete subtree."""
    if world == 1:
        return True
    if world & (world - 1):
        return False
    segs = [(0, total)]
    while len(segs) < world:
        nxt = []
        for off, ln in segs:
            if ln <= 128:
                return False
            n2 = ln // 2
            n2 -= n2 % 8
            nxt += [(off, n2), (off + n2, ln - n2)]
        segs = nxt
    blk = total // world
    return all(off == k * blk and ln == blk for k, (off, ln) in enumerate(segs))


def combine_subtrees(parts: list[float]) -> float:
    """Top of the pairwise tree over power-of-two aligned subtrees."""
    if len(parts) == 1:
        return parts[0]
    h = len(parts) // 2
    return combine_subtrees(parts[:h]) + combine_subtrees(parts[h:])


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------
class Comm:
    """torch.distributed collectives on the ops' tensors (NCCL on GPU, gloo on CPU)."""

    def __init__(self):
        import torch.distributed as dist

        self.dist = dist
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()

    def send(self, t, dst: int) -> None:
        self.dist.send(t.contiguous(), dst)

    def recv_like(self, like, src: int):
        import torch

        t = torch.empty_like(like)
        self.dist.recv(t, src)
        return t

    def broadcast(self, t, src: int):
        t = t.contiguous()
        self.dist.broadcast(t, src)
        return t

    def all_reduce_sum(self, t):
        t = t.contiguous()
        self.dist.all_reduce(t)
        return t

    def all_gather_cat(self, t):
        """Concatenate equally shaped per-rank tensors along dim 0, in rank order."""
        import torch

        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t.contiguous())
        return torch.cat(parts, dim=0)

    def all_max(self, v: int) -> int:
        import torch

        t = torch.tensor([int(v)], dtype=torch.int64)
        if self.dist.get_backend() == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return int(t.item())


class SingleComm:
    """World of one (no process group)."""

    world = 1
    rank = 0

    def send(self, t, dst):  # pragma: no cover - never called with world 1
        raise RuntimeError("send in a world of one")

    recv_like = send

    def broadcast(self, t, src):
        return t

    def all_reduce_sum(self, t):
        return t

    def all_gather_cat(self, t):
        return t

    def all_max(self, v):
        return int(v)


# ---------------------------------------------------------------------------
# device operations through the C ABI
# ---------------------------------------------------------------------------
class GpuOps:
    """Phase operations on CUDA tensors; quaternion matrices are (rows, cols, 4) float64."""

    def __init__(self, dev=None):
        self.dev = dev or _native.device()
        self.torch = self.dev.torch

    def vec(self, n):
        return self.dev.empty(int(n))

    def colsums_seq(self, xb, acc):
        rows, n = int(xb.shape[0]), int(xb.shape[1])
        sq = self.dev.empty(rows * n)
        col = self.dev.empty(n)
        self.dev.call("qcur_colsums_seq", xb.data_ptr(), rows, n, 0 if acc is None else acc.data_ptr(),
                      col.data_ptr(), sq.data_ptr())
        return sq, col

    def colsums_chunk(self, xb, c0, c1, acc, colsum, sq):
        """Columns [c0, c1) of the sequential chain: colsum[c0:c1] and sq[:, c0:c1] (row pitch n)."""
        rows, n = int(xb.shape[0]), int(xb.shape[1])
        self.dev.call("qcur_colsums_seq_ex", xb.data_ptr() + 32 * c0, rows, c1 - c0, n,
                      0 if acc is None else acc.data_ptr(), colsum.data_ptr() + 8 * c0, sq.data_ptr() + 8 * c0, n)

    def pairwise(self, data, nseg, length):
        out = self.dev.empty(int(nseg))
        self.dev.call("qcur_pairwise_sums", data.data_ptr(), int(nseg), int(length), int(length), out.data_ptr())
        return out

    def div(self, v, denom):
        d = self.torch.tensor([float(denom)], dtype=self.torch.float64, device=v.device) \
            if not hasattr(denom, "data_ptr") else denom
        out = self.dev.empty(int(v.numel()))
        self.dev.call("qcur_vec_div", v.data_ptr(), int(v.numel()), d.data_ptr(), out.data_ptr())
        return out

    def scalar(self, t) -> float:
        return float(t.reshape(-1)[0].item())

    def uniform(self, m, n):
        col, row = self.vec(n), self.vec(m)
        self.dev.call("qcur_uniform_distributions", int(m), int(n), col.data_ptr(), row.data_ptr())
        return col, row

    def draw(self, probs, count, state):
        out = self.dev.empty(int(count), dtype=self.torch.int64)
        self.dev.call("qcur_draw_indices", probs.data_ptr(), int(probs.numel()), int(count),
                      state.ctypes.data_as(_native._u64p), out.data_ptr())
        return out

    def gather_cols(self, xb, J):
        rows, n = int(xb.shape[0]), int(xb.shape[1])
        out = self.dev.empty_q(rows, int(J.numel()))
        self.dev.call("qcur_gather_cols", xb.data_ptr(), rows, n, J.data_ptr(), int(J.numel()), out.data_ptr())
        return out

    def gather_rows(self, xb, local_rows):
        n = int(xb.shape[1])
        k = int(local_rows.numel())
        out = self.dev.empty_q(max(k, 1), n)
        if k:
            self.dev.call("qcur_gather_rows", xb.data_ptr(), n, local_rows.data_ptr(), k, out.data_ptr())
        return out[:k]

    def index_tensor(self, values):
        return self.torch.tensor(list(values), dtype=self.torch.int64, device=f"cuda:{self.dev.index}")

    def to_host_int(self, t) -> np.ndarray:
        return t.cpu().numpy()

    def gemm(self, A, B, opA=0, opB=0, alpha=1.0, flags=0):
        M = int(A.shape[1] if opA else A.shape[0])
        K = int(A.shape[0] if opA else A.shape[1])
        N = int(B.shape[0] if opB else B.shape[1])
        out = self.dev.empty_q(M, N)
        self.dev.call("qcur_qgemm_ex", opA, opB, M, N, K, float(alpha), A.data_ptr(), int(A.shape[1]), B.data_ptr(),
                      int(B.shape[1]), 0.0, out.data_ptr(), N, int(flags))
        return out

    def xq(self, xb, QR):
        rows, n, r = int(xb.shape[0]), int(xb.shape[1]), int(QR.shape[1])
        out = self.dev.empty_q(rows, r)
        self.dev.call("qcur_xq", xb.data_ptr(), rows, n, n, QR.data_ptr(), r, out.data_ptr())
        return out

    def chol_inv(self, G):
        q = int(G.shape[0])
        out = self.dev.empty_q(q, q)
        self.dev.call("qcur_chol_inv", G.data_ptr(), q, out.data_ptr())
        return out

    def series(self, G2):
        q = int(G2.shape[0])
        out = self.dev.empty_q(q, q)
        self.dev.call("qcur_series_l2inv", G2.data_ptr(), q, out.data_ptr())
        return out

    def series_inv(self, G2):
        q = int(G2.shape[0])
        out = self.dev.empty_q(q, q)
        self.dev.call("qcur_series_inv", G2.data_ptr(), q, out.data_ptr())
        return out

    def kappa(self, G1, F):
        self.dev.call("qcur_kappa_check", G1.data_ptr(), F.data_ptr(), int(G1.shape[0]))

    def fast_failed(self) -> bool:
        self.dev.call("qcur_check")
        return bool(self.dev.info() & 4)

    def factor(self, Z, zh):
        p = int(Z.shape[0] if not zh else Z.shape[1])
        q = int(Z.shape[1] if not zh else Z.shape[0])
        Q, F = self.dev.empty_q(p, q), self.dev.empty_q(q, q)
        self.dev.call("qcur_factor", Z.data_ptr(), int(zh), p, q, Q.data_ptr(), F.data_ptr())
        return Q, F

    def error_stats(self, xb, Cb, U, R, psnr_scale=0.0):
        rows, n = int(xb.shape[0]), int(xb.shape[1])
        out4 = self.dev.empty(4)
        self.dev.call("qcur_cur_error", xb.data_ptr(), rows, n, Cb.data_ptr(), int(Cb.shape[1]), U.data_ptr(),
                      R.data_ptr(), int(R.shape[0]), float(psnr_scale), out4.data_ptr())
        return out4

    def stack_stats(self, t):
        return t.reshape(1, 4)


# ---------------------------------------------------------------------------
# the sharded approximation
# ---------------------------------------------------------------------------
def approx_rowsharded(ops, comm, xb, m: int, strategy: str, seed: int, c: int, r: int,
                      psnr_scale: float = 0.0) -> dict:
    """One QMCUR approximation of the m x n matrix whose row block `xb`
    (rows [rank*m/G, (rank+1)*m/G)) this rank holds.  Returns the replicated
    J, I, U, R, the local C rows and the global error statistics."""
    G, g = comm.world, comm.rank
    rows_b, n = int(xb.shape[0]), int(xb.shape[1])
    if rows_b * G != m:
        raise ValueError("row-block sharding needs m divisible by the world size")
    row0 = g * rows_b
    # ---- K1: sampling distributions -------------------------------------
    if strategy == "length":
        if not subtree_aligned(m * n, G):
            raise NotImplementedError(
                f"numpy's pairwise tree over {m}x{n} does not split at the row blocks of {G} ranks")
        # numpy's sequential column chain continued rank to rank, pipelined by column chunks: rank
        # g works on chunk k as soon as rank g-1 has passed it on (a wavefront: G + K - 1 chunk
        # times instead of G whole passes)
        nchunks = 1 if G == 1 else max(1, min(4 * G, n // 64))
        bounds = [n * k // nchunks for k in range(nchunks + 1)]
        sq, colsum = ops.vec(rows_b * n), ops.vec(n)
        for k in range(nchunks):
            c0, c1 = bounds[k], bounds[k + 1]
            acc = None if g == 0 else comm.recv_like(ops.vec(c1 - c0), g - 1)
            ops.colsums_chunk(xb, c0, c1, acc, colsum, sq)
            if g < G - 1:
                comm.send(colsum[c0:c1], g + 1)
        colsum = comm.broadcast(colsum, G - 1)
        rowsum = ops.pairwise(sq, rows_b, n)
        part = ops.pairwise(sq, 1, rows_b * n)
        parts = comm.all_gather_cat(part)
        total = combine_subtrees([float(v) for v in parts.cpu().numpy()])
        if not total > 0.0:
            from .errors import DegenerateDistributionError

            raise DegenerateDistributionError("all sampling weights vanish (zero matrix)")
        col = ops.div(colsum, total)
        rowp = comm.all_gather_cat(ops.div(rowsum, total))
        colp = ops.div(col, ops.scalar(ops.pairwise(col, 1, n)))
        rowp = ops.div(rowp, ops.scalar(ops.pairwise(rowp, 1, m)))
    else:
        colp, rowp = ops.uniform(m, n)
    # ---- K2: identical draws everywhere ----------------------------------
    st = _native.state_from_seed(seed)
    J = ops.draw(colp, c, st)  # advances st by c
    I = ops.draw(rowp, r, st)
    # ---- K3: C rows local; R rows by owner + all-gather (byte copies) -----
    Cb = ops.gather_cols(xb, J)
    I_host = ops.to_host_int(I)
    owned = [t for t in range(r) if row0 <= int(I_host[t]) < row0 + rows_b]
    kmax = comm.all_max(len(owned))
    Rown = ops.gather_rows(xb, ops.index_tensor([int(I_host[t]) - row0 for t in owned]))
    import torch

    buf = torch.zeros((kmax, n, 4), dtype=torch.float64, device=Rown.device)
    buf[: len(owned)] = Rown
    allrows = comm.all_gather_cat(buf)  # (G*kmax, n, 4): owner g's rows at [g*kmax, g*kmax + #owned_g)
    # one device gather puts row t of R (drawn index I[t]) in place: its slot in the gathered
    # buffer is (owner of I[t]) * kmax + (its rank among that owner's draws, in draw order)
    slot = np.empty(r, dtype=np.int64)
    seen = np.zeros(G, dtype=np.int64)
    for t in range(r):
        owner = int(I_host[t]) // rows_b
        slot[t] = owner * kmax + seen[owner]
        seen[owner] += 1
    R = ops.gather_rows(allrows, ops.index_tensor(slot))
    # ---- K4: pinv(C) by distributed CholeskyQR2, pinv(R) replicated ------
    G1 = comm.all_reduce_sum(ops.gemm(Cb, Cb, opA=1, flags=2))
    X1 = ops.chol_inv(G1)
    Q1 = ops.gemm(Cb, X1, opB=1, flags=1)
    G2 = comm.all_reduce_sum(ops.gemm(Q1, Q1, opA=1, flags=2))
    # as the monolithic factor (qcur_abi.cu factor_multi): pinv(C) = F Q1^H with
    # F = L1^-H G2^-1 = L1^-H (I - E + E^2), E = G2 - I; the kappa guard on ||L1^-1||_F
    QC = Q1
    S = ops.series_inv(G2)
    ops.kappa(G1, X1)
    FC = ops.gemm(X1, S, opA=1)
    failed = ops.fast_failed()
    if comm.all_max(1 if failed else 0):  # robust path: factor the gathered C locally
        Cfull = comm.all_gather_cat(Cb)
        QCfull, FC = ops.factor(Cfull, 0)
        QC = QCfull[row0:row0 + rows_b]
    QR, FR = ops.factor(R, 1)
    # ---- K6/K7: U ----------------------------------------------------------
    Yb = ops.xq(xb, QR)  # the big contraction on qmcur's engine (INT8 tensor cores when large)
    M = comm.all_reduce_sum(ops.gemm(QC, Yb, opA=1))
    U = ops.gemm(ops.gemm(FC, M), FR, opB=1)
    # ---- K8/K9: fused error, partials in rank order -------------------------
    stats = comm.all_gather_cat(ops.stack_stats(ops.error_stats(xb, Cb, U, R, psnr_scale)))
    tot = [0.0, 0.0, 0.0, 0.0]
    for row in stats.cpu().numpy():
        for k in range(4):
            tot[k] += float(row[k])
    return dict(J=J, I=I, Cb=Cb, U=U, R=R, stats=tot, rel_err=math.sqrt(tot[0]) / math.sqrt(tot[1]))
