"""Row-sharded 2-D 5-point stencil across ranks (one process per GPU).

BASELINE config 4 / SURVEY.md §8(e): the grid's rows are split into
contiguous slabs, one per rank; each slab carries `ghost` rows above and
below.  One temporal block of depth bt reads the bt ghost rows on each side
(the trapezoid shrinks by one row per step), so every bt steps each rank
sends its first/last bt owned rows to its neighbours' ghost rows — the
only data exchange.  The exchange is overlapped with compute: the boundary
strips (rows [0, bt) and [R-bt, R)) are advanced first on one stream, their
sends/recvs (torch.distributed, NCCL on GPUs) start as soon as they finish,
and the interior rows are advanced concurrently on a second stream.

The reference has no distributed path; results must equal the
single-grid run bit for bit, which the per-point arithmetic guarantees as
long as the ghost rows hold the neighbour's step-t0 values.

The slab kernel is injected (`advance`) so the same exchange logic — the
same edge-strips-first / post sends / interior / wait sequence, line for
line — runs with the sm_100a kernel on GPUs and with a CPU restatement under
gloo in the tests; on CPU the "streams" are no-op lanes.

halo="p2p" fuses the exchange into the stencil kernel instead: both slabs
live in symmetric memory (torch.distributed._symmetric_memory, peer buffers
mapped over NVLink), one launch per block advances every owned row and
stores its first/last bt output rows a second time, straight into the
neighbours' ghost rows (`pcotgpu_s2d5_advance_p2p`); a device-side barrier on
the stream then orders the block against the neighbours' next one.  No
send/recv, no separate edge launches.  The fused kernel and the barrier are
injectable too (`advance_p2p`, `barrier`, `buffers`), so the ordering logic
runs on CPU with the mirror stores emulated into shared-memory buffers.
"""
import contextlib
import ctypes

import torch
import torch.distributed as dist

import paper_1802_00166_b200 as P


def mirror_targets(peer_out_origin_up, peer_out_origin_dn, rows, ld, elem=8):
    """Addresses the P2P kernel takes as mirror_up / mirror_dn: output row r of
    this slab lands at mirror + (r*ld + col)*elem, i.e. the upper neighbour's
    row R + r (its ghost rows below, r < bt) and the lower neighbour's row r - R
    (its ghost rows above, r >= R - bt).  None = no neighbour on that side.
    elem=8: byte addresses (the kernel); elem=1: element offsets (emulation)."""
    up = None if peer_out_origin_up is None else peer_out_origin_up + rows * ld * elem
    dn = None if peer_out_origin_dn is None else peer_out_origin_dn - rows * ld * elem
    return up, dn


def layout(rows, cols):
    ld, ghost, padl, total = (ctypes.c_int64() for _ in range(4))
    P._check(P.lib().pcotgpu_s2d5_layout(rows, cols, ctypes.byref(ld), ctypes.byref(ghost),
                                         ctypes.byref(padl), ctypes.byref(total)))
    return ld.value, ghost.value, padl.value, total.value


class ShardedStencil2D:
    """One rank's slab of an (R * world) x cols grid; ring rows/cols are the
    global grid's edges (ring_hold=0: literal 0.0, 1: copied forward)."""

    def __init__(self, rows_per_rank, cols, T, bt, ring_hold=0, order=0, device=None,
                 advance=None, geometry=None, group=None, halo="nccl", advance_p2p=None,
                 barrier=None, buffers=None):
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.group = group
        self.R, self.cols, self.T, self.bt = int(rows_per_rank), int(cols), int(T), int(bt)
        self.ring_hold, self.order = int(ring_hold), int(order)
        self.g0 = self.rank * self.R
        self.nrows = self.R * self.world
        if self.R < 2 * self.bt and self.world > 1:
            raise ValueError("slab must hold at least 2*bt rows")
        self.device = device if device is not None else torch.device("cpu")
        if geometry is None:
            geometry = layout(self.R, self.cols)
        self.ld, self.ghost, self.padl, total = geometry
        if self.ghost < self.bt + 3:
            raise ValueError("ghost rows < bt + 3")
        self.on_gpu = self.device.type == "cuda"
        if halo not in ("nccl", "p2p"):
            raise ValueError("halo must be 'nccl' or 'p2p'")
        # (at world size 1 the symmetric-memory path still runs: no neighbours,
        # so no mirror stores, but the allocation, rendezvous and barrier do)
        self.p2p = halo == "p2p"
        emulated = advance_p2p is not None and barrier is not None and buffers is not None
        if self.p2p and not emulated and not (self.on_gpu and dist.is_initialized()):
            raise ValueError("halo='p2p' needs CUDA devices and an initialised process group")
        if buffers is not None:  # caller-owned slabs (the P2P emulation's shared memory)
            self.buf = list(buffers)
        elif self.p2p:
            from torch.distributed import _symmetric_memory as symm

            grp = self.group if self.group is not None else dist.group.WORLD
            self.buf, self.symm = [], []
            for _ in range(2):
                t = symm.empty(total, dtype=torch.float64, device=self.device)
                t.zero_()
                self.buf.append(t)
                self.symm.append(symm.rendezvous(t, grp))
        else:
            self.buf = [torch.zeros(total, dtype=torch.float64, device=self.device) for _ in range(2)]
        self.cur = 0
        self.advance = advance or self._advance_cuda
        self.advance_p2p = advance_p2p or self._advance_p2p
        self.barrier = barrier or (lambda b: self.symm[b].barrier(channel=0))
        if self.on_gpu:
            self.s_edge = torch.cuda.Stream(device=self.device, priority=-1)
            self.s_inner = torch.cuda.Stream(device=self.device)
        self.kernel_events = []  # (start, end) CUDA events of every slab launch when timing

    # -------------------------------------------------------------- views
    def origin_offset(self):
        return self.ghost * self.ld + self.padl

    def rows_view(self, b, r0, r1):
        """Flat contiguous view of local rows [r0, r1) (full pitch) of buffer b."""
        base = (self.ghost + r0) * self.ld
        return self.buf[b][base:base + (r1 - r0) * self.ld]

    def interior(self, b):
        """(R, cols) strided view of the owned cells of buffer b."""
        v = self.buf[b][self.ghost * self.ld:(self.ghost + self.R) * self.ld].view(self.R, self.ld)
        return v[:, self.padl:self.padl + self.cols]

    def ptr(self, b):
        return self.buf[b].data_ptr() + self.origin_offset() * 8

    # -------------------------------------------------------------- init
    def fill_init(self, name="F"):
        """F[g, c] = init_value(name, g*cols + c) on owned rows, ring applied."""
        b = self.cur
        if self.on_gpu:
            s = torch.cuda.current_stream(self.device)
            P._check(P.lib().pcotgpu_fill_init_value(
                ctypes.c_void_p(self.ptr(b)), self.ld, self.R, self.cols, name.encode(),
                self.g0 * self.cols, ctypes.c_void_p(s.cuda_stream)))
            P._check(P.lib().pcotgpu_s2d5_prepare(
                ctypes.c_void_p(self.ptr(b)), self.R, self.cols, self.g0, self.nrows,
                self.ring_hold, ctypes.c_void_p(s.cuda_stream)))
        else:
            raise RuntimeError("fill_init needs the GPU library; load values with load()")
        self.exchange_sync(b)

    def snapshot_input(self):
        """Keep the step-0 slab (owned + ghost rows) so every run restarts from F,
        as the reference's init statement re-reads F on every run."""
        self.f0 = self.buf[self.cur].clone()

    def restart(self):
        self.buf[0].copy_(self.f0)
        self.cur = 0

    def load(self, values):
        """Owned rows from a (R, cols) tensor (any device); ghosts from neighbours."""
        self.interior(self.cur).copy_(values)
        self.exchange_sync(self.cur)

    # -------------------------------------------------------------- exchange
    def _ops(self, b, depth):
        ops = []
        up, dn = self.rank - 1, self.rank + 1
        g = self.group
        if up >= 0:
            ops.append(dist.P2POp(dist.isend, self.rows_view(b, 0, depth), up, g))
            ops.append(dist.P2POp(dist.irecv, self.rows_view(b, -depth, 0), up, g))
        if dn < self.world:
            ops.append(dist.P2POp(dist.isend, self.rows_view(b, self.R - depth, self.R), dn, g))
            ops.append(dist.P2POp(dist.irecv, self.rows_view(b, self.R, self.R + depth), dn, g))
        return ops

    def exchange_sync(self, b, depth=None):
        if self.world == 1:
            return
        depth = depth or min(self.ghost, self.R)
        ops = self._ops(b, depth)
        for r in dist.batch_isend_irecv(ops):
            r.wait()

    # -------------------------------------------------------------- compute
    def _advance_cuda(self, src, dst, row_lo, row_hi, bt, stream):
        P._check(P.lib().pcotgpu_s2d5_advance(
            ctypes.c_void_p(self.ptr(src)), ctypes.c_void_p(self.ptr(dst)), self.R, self.cols,
            self.g0, self.nrows, bt, self.ring_hold, self.order, row_lo, row_hi,
            ctypes.c_void_p(stream.cuda_stream if stream is not None else 0)))

    def _peer_origin(self, b, peer):
        if peer < 0 or peer >= self.world:
            return None
        return int(self.symm[b].buffer_ptrs[peer]) + self.origin_offset() * 8

    def _advance_p2p(self, src, dst, bt, stream):
        up, dn = mirror_targets(self._peer_origin(dst, self.rank - 1),
                                self._peer_origin(dst, self.rank + 1), self.R, self.ld)
        P._check(P.lib().pcotgpu_s2d5_advance_p2p(
            ctypes.c_void_p(self.ptr(src)), ctypes.c_void_p(self.ptr(dst)), self.R, self.cols,
            self.g0, self.nrows, bt, self.ring_hold, self.order, 0, self.R,
            ctypes.c_void_p(up), ctypes.c_void_p(dn), bt, ctypes.c_void_p(stream.cuda_stream)))

    def _timed(self, fn, stream, record):
        if record and self.on_gpu:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            self.kernel_events.append((e0, e1))
        else:
            fn()

    # lanes: CUDA streams on the GPU; on CPU the same sequence with no-op lanes
    def _main(self):
        return torch.cuda.current_stream(self.device) if self.on_gpu else None

    def _on(self, lane):
        return torch.cuda.stream(lane) if lane is not None else contextlib.nullcontext()

    def _fork(self):
        if not self.on_gpu:
            return None, None
        main = self._main()
        self.s_edge.wait_stream(main)
        self.s_inner.wait_stream(main)
        return self.s_edge, self.s_inner

    def _join(self):
        if self.on_gpu:
            main = self._main()
            main.wait_stream(self.s_edge)
            main.wait_stream(self.s_inner)

    def block(self, bt, record=False):
        """Advance all owned rows by bt steps, exchanging boundary rows."""
        src, dst = self.cur, self.cur ^ 1
        if self.world == 1 and not self.p2p:
            main = self._main()
            self._timed(lambda: self.advance(src, dst, 0, self.R, bt, main), main, record)
        elif self.p2p:
            # one launch: owned rows + their mirror stores into the neighbours'
            # ghost rows of `dst`; the barrier (after this kernel, on the same
            # stream) waits for the neighbours' kernels of this block, whose
            # stores filled our ghost rows, before anyone starts the next block
            main = self._main()
            self._timed(lambda: self.advance_p2p(src, dst, bt, main), main, record)
            self.barrier(dst)
        else:
            # overlapped NCCL exchange: boundary strips first, their rows go out
            # while the interior is advanced on the other lane; the receives
            # complete before the next block reads the ghost rows
            edge, inner = self._fork()
            e = self.bt if self.R >= 2 * self.bt else self.R
            with self._on(edge):
                self._timed(lambda: self.advance(src, dst, 0, e, bt, edge), edge, record)
                self._timed(lambda: self.advance(src, dst, self.R - e, self.R, bt, edge), edge, record)
                reqs = dist.batch_isend_irecv(self._ops(dst, bt))
            with self._on(inner):
                self._timed(lambda: self.advance(src, dst, e, self.R - e, bt, inner), inner, record)
            with self._on(edge):
                for r in reqs:
                    r.wait()
            self._join()
        self.cur = dst

    def run(self, record=False):
        """T steps in blocks of bt (last block shorter)."""
        t = 0
        while t < self.T:
            step = min(self.bt, self.T - t)
            self.block(step, record)
            t += step

    def launches_per_run(self):
        blocks = -(-self.T // self.bt)
        return blocks * (1 if self.world == 1 or self.p2p else 3)
