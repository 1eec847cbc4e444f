"""Training-step mirror (include/sxen/trainer.hpp, src/trainer.cpp) over sxen_trainer_*.

``train_field`` follows the reference's contract: a BatchSampler fills (coords, aux, targets) for each step, the step
runs encode -> forward -> MSE -> backward -> encode_backward, then sparse Adam on the tables and dense Adam on the MLP.
With ``world_size > 1`` (torch.distributed initialised) each rank takes its contiguous chunk of the batch exactly as the
reference's workers do (src/trainer.cpp:93,107-108) and the gradient buffers are all-reduced where the reference merges
its per-worker accumulators (:125-128)."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, List, Tuple

from . import _abi
from .errors import TrainingError, raise_for
from .optimizer import AdamConfig


def _lib():
    from . import lib
    return lib


@dataclass
class TrainConfig:
    """sxen::TrainConfig, same defaults (include/sxen/trainer.hpp:15-24).  `threads` has no device meaning."""

    batch_size: int = 2048
    steps: int = 10000
    aux_dims: int = 0
    table_adam: AdamConfig = field(default_factory=lambda: AdamConfig(lr=1e-2, beta1=0.9, beta2=0.99, epsilon=1e-15))
    mlp_adam: AdamConfig = field(default_factory=lambda: AdamConfig(lr=1e-3, beta1=0.9, beta2=0.99, epsilon=1e-15))
    seed: int = 1234
    threads: int = 0
    record_every: int = 100
    reproducible: bool = False  # no reference field: order-free gradient sums (Trainer.set_reproducible)


@dataclass
class TrainResult:
    loss_curve: List[Tuple[int, float]] = field(default_factory=list)
    final_loss: float = 0.0
    steps_run: int = 0


def chunk_bounds(batch: int, workers: int, worker: int) -> Tuple[int, int]:
    """The reference's contiguous chunking (src/trainer.cpp:93,107-108): chunk = ceil(B/T), worker t takes
    [t*chunk, min(B, (t+1)*chunk)).  Ranks play the workers."""
    chunk = (batch + workers - 1) // workers
    begin = min(batch, worker * chunk)
    return begin, min(batch, begin + chunk)


class Trainer:
    """Owns the gradient accumulator and both Adam states for one (encoder, mlp) pair."""

    def __init__(self, encoder, mlp, aux_dims: int = 0):
        """aux_dims: TrainConfig::aux_dims, extra inputs per sample appended after the encoding (src/trainer.cpp:32-35);
        the MLP's input width must be encoded width + aux_dims (ValueError otherwise, :61-65)."""
        self._lib = _lib()
        self._h = C.c_void_p()
        self.encoder, self.mlp, self.aux_dims = encoder, mlp, int(aux_dims)
        self._aux = None
        raise_for(self._lib, self._lib.sxen_trainer_create_aux(encoder._h, mlp._h, int(aux_dims), C.byref(self._h)))

    def set_aux(self, aux) -> None:
        """The [batch, aux_dims] CUDA tensor (f64 or f32) the next accumulate / step calls read; kept alive here."""
        if aux is None:
            self._aux = None
            raise_for(self._lib, self._lib.sxen_trainer_set_aux(self._h, None, _abi.COORD_F64))
            return
        aux = aux.contiguous()
        if aux.dim() != 2 or aux.shape[1] != self.aux_dims:
            raise ValueError(f"train: aux must be [batch, {self.aux_dims}]")
        self._aux = aux
        raise_for(self._lib, self._lib.sxen_trainer_set_aux(self._h, C.c_void_p(aux.data_ptr()), self._typ(aux)))

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.sxen_trainer_destroy(self._h)
            self._h = None

    @staticmethod
    def _typ(t):
        import torch
        return {torch.float64: _abi.COORD_F64, torch.float32: _abi.COORD_F32}[t.dtype]

    def accumulate(self, coords, targets, global_batch: int, stream=None) -> None:
        from .encoding import _stream_ptr
        coords, targets = coords.contiguous(), targets.contiguous()
        raise_for(self._lib, self._lib.sxen_trainer_accumulate(
            self._h, C.c_void_p(coords.data_ptr()), self._typ(coords), C.c_void_p(targets.data_ptr()),
            self._typ(targets), coords.shape[0], global_batch, _stream_ptr(stream, self.encoder.device)))

    def accumulate_head(self, coords, targets, global_batch: int, stream=None) -> None:
        """encode -> MLP forward -> loss/upstream -> MLP backward; d(loss)/d(encoding) stays in the workspace."""
        from .encoding import _stream_ptr
        raise_for(self._lib, self._lib.sxen_trainer_accumulate_head(
            self._h, C.c_void_p(coords.data_ptr()), self._typ(coords), C.c_void_p(targets.data_ptr()),
            self._typ(targets), coords.shape[0], global_batch, _stream_ptr(stream, self.encoder.device)))

    def accumulate_tables(self, coords, first_level: int, level_count: int, stream=None) -> None:
        """encode_backward of the batch of the last accumulate_head for one range of encoder levels."""
        from .encoding import _stream_ptr
        raise_for(self._lib, self._lib.sxen_trainer_accumulate_tables(
            self._h, C.c_void_p(coords.data_ptr()), self._typ(coords), coords.shape[0], first_level, level_count,
            _stream_ptr(stream, self.encoder.device)))

    def table_grad_device(self):
        """Flat float32 view of the table-gradient accumulator (untouched rows carry -0.0; SUM all-reduce keeps that)."""
        import torch
        from .encoding import _wrap_device
        g = C.c_void_p()
        raise_for(self._lib, self._lib.sxen_trainer_table_grad(self._h, C.byref(g)))
        ptr, cnt = C.c_void_p(), C.c_size_t()
        raise_for(self._lib, self._lib.sxen_grad_values_dev(g, C.byref(ptr), C.byref(cnt)))
        return _wrap_device(ptr.value, cnt.value, torch.float32, self)

    def table_grad_fixed_device(self):
        """The accumulator's fixed-point words (flat int64 view) in reproducible mode, else None; summed over the ranks
        next to the f32 values, which then only carry the touched markers."""
        import torch
        from .encoding import _DevArray
        g = C.c_void_p()
        raise_for(self._lib, self._lib.sxen_trainer_table_grad(self._h, C.byref(g)))
        ptr, cnt = C.c_void_p(), C.c_size_t()
        raise_for(self._lib, self._lib.sxen_grad_fixed_dev(g, C.byref(ptr), C.byref(cnt)))
        if not ptr.value:
            return None
        return torch.as_tensor(_DevArray(ptr.value, cnt.value, "<i8", self), device=f"cuda:{self.encoder.device}")

    def loss_device(self):
        import torch
        from .encoding import _wrap_device
        p = C.c_void_p()
        raise_for(self._lib, self._lib.sxen_trainer_loss_dev(self._h, C.byref(p)))
        return _wrap_device(p.value, 1, torch.float64, self)

    def loss(self, global_batch: int, stream=None) -> float:
        from .encoding import _stream_ptr
        out = C.c_double()
        raise_for(self._lib, self._lib.sxen_trainer_loss(self._h, global_batch, C.byref(out), _stream_ptr(stream, self.encoder.device)))
        return out.value

    def update(self, table_adam: AdamConfig, mlp_adam: AdamConfig, stream=None, check: bool = True) -> None:
        from .encoding import _stream_ptr
        ta, ma = table_adam.c(), mlp_adam.c()
        raise_for(self._lib, self._lib.sxen_trainer_update(self._h, C.byref(ta), C.byref(ma), _stream_ptr(stream, self.encoder.device)))
        if check:
            raise_for(self._lib, self._lib.sxen_trainer_check(self._h, _stream_ptr(stream, self.encoder.device)))

    def step(self, coords, targets, table_adam: AdamConfig, mlp_adam: AdamConfig, stream=None) -> float:
        """One whole single-GPU step; returns the batch MSE before the update (TrainResult::loss_curve's value)."""
        from .encoding import _stream_ptr
        coords, targets = coords.contiguous(), targets.contiguous()
        ta, ma = table_adam.c(), mlp_adam.c()
        out = C.c_double()
        raise_for(self._lib, self._lib.sxen_trainer_step(
            self._h, C.c_void_p(coords.data_ptr()), self._typ(coords), C.c_void_p(targets.data_ptr()),
            self._typ(targets), coords.shape[0], C.byref(ta), C.byref(ma), C.byref(out), _stream_ptr(stream, self.encoder.device)))
        return out.value

    def step_enqueue(self, coords, targets, table_adam: AdamConfig, mlp_adam: AdamConfig, stream=None) -> None:
        """Queues one whole step (gradient pass, loss into the device ring, both updates) without waiting for it;
        ``collect`` returns the losses.  A non-finite loss stops every later update on the device."""
        from .encoding import _stream_ptr
        coords, targets = coords.contiguous(), targets.contiguous()
        ta, ma = table_adam.c(), mlp_adam.c()
        raise_for(self._lib, self._lib.sxen_trainer_step_enqueue(
            self._h, C.c_void_p(coords.data_ptr()), self._typ(coords), C.c_void_p(targets.data_ptr()),
            self._typ(targets), coords.shape[0], C.byref(ta), C.byref(ma), _stream_ptr(stream, self.encoder.device)))

    def pending(self) -> int:
        n = C.c_size_t()
        raise_for(self._lib, self._lib.sxen_trainer_pending(self._h, C.byref(n)))
        return n.value

    def collect(self, stream=None):
        """(losses, failed): the losses of the steps queued since the last collect; ``failed`` is the index of the
        first non-finite one (the updates from that step on were not applied) or -1.  Rejected samples and non-finite
        gradients raise like ``step``."""
        from . import _abi
        from .encoding import _stream_ptr
        n = self.pending()
        buf = (C.c_double * max(n, 1))()
        cnt, failed = C.c_size_t(), C.c_int64(-1)
        st = self._lib.sxen_trainer_collect(self._h, buf, n, C.byref(cnt), C.byref(failed), _stream_ptr(stream, self.encoder.device))
        if st == _abi.TRAINING_ERROR and failed.value >= 0:
            return list(buf[:cnt.value]), failed.value
        raise_for(self._lib, st)
        return list(buf[:cnt.value]), -1

    def set_fused(self, mode: int = 0) -> None:
        """sxen_trainer_set_fused: 0 = three kernels (default, measured faster), 1 = the one-kernel step (encode -> tcgen05
        head -> encode_backward, nothing through HBM) or ValueError, -1 = fused whenever the shapes allow."""
        raise_for(self._lib, self._lib.sxen_trainer_set_fused(self._h, int(mode)))

    def set_reproducible(self, on: bool = True) -> None:
        """sxen_trainer_set_reproducible: bit-reproducible steps (order-free fixed-point gradient sums for the tables and
        the MLP; with the exact head d(loss)/d(encoding) reaches encode_backward as doubles)."""
        raise_for(self._lib, self._lib.sxen_trainer_set_reproducible(self._h, 1 if on else 0))

    def set_comm(self, comm) -> None:
        """Attaches a ``Comm`` (kept alive here; None detaches): ``step_sharded`` then exchanges through the C ABI."""
        self._comm_handle = comm
        raise_for(self._lib, self._lib.sxen_trainer_set_comm(self._h, comm._h if comm is not None else None))

    def step_sharded(self, coords, targets, table_adam: AdamConfig, mlp_adam: AdamConfig, level_chunks: int = 4,
                     stream=None) -> float:
        """sxen_trainer_step_sharded: one whole batch-sharded step inside the library -- coords / targets hold the WHOLE batch
        on every rank, this rank runs its contiguous chunk (src/trainer.cpp:93,107-108), the exchange (the attached Comm)
        overlaps the backward level range by level range, every rank applies the identical update.  Returns the batch MSE
        before the update; raises TrainingError (nothing updated, on any rank) when it is non-finite."""
        from .comm import _check
        from .encoding import _stream_ptr
        coords, targets = coords.contiguous(), targets.contiguous()
        ta, ma = table_adam.c(), mlp_adam.c()
        out = C.c_double()
        _check(self._lib, self._lib.sxen_trainer_step_sharded(
            self._h, C.c_void_p(coords.data_ptr()), self._typ(coords), C.c_void_p(targets.data_ptr()), self._typ(targets),
            coords.shape[0], C.byref(ta), C.byref(ma), level_chunks, C.byref(out), _stream_ptr(stream, self.encoder.device)))
        return out.value

    def distributed_step(self, coords, targets, table_adam: AdamConfig, mlp_adam: AdamConfig, group=None,
                         level_chunks: int = 4) -> float:
        """Batch-sharded step: coords/targets hold the WHOLE batch on every rank (the sampler is deterministic in
        (seed, step), so no scatter is needed); this rank runs its contiguous chunk, then table gradients, MLP gradients
        and the loss sum are all-reduced (SUM) and every rank applies the identical update.

        The exchange overlaps the backward: after the MLP half, encode_backward walks the levels in ``level_chunks``
        ranges; each range's slice of the accumulator (contiguous, level-major) is all-reduced on a second stream while
        the next range computes.  The MLP gradient and the loss sum go first, under the first range."""
        import torch
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        batch = coords.shape[0]
        b, e = chunk_bounds(batch, world, rank)
        x, t = coords[b:e].contiguous(), targets[b:e].contiguous()
        levels = self.encoder.config.levels
        bounds = level_ranges(levels, level_chunks)
        gview = self.table_grad_device()
        fview = self.table_grad_fixed_device()
        per_level = gview.numel() // levels
        if not x.is_cuda:
            raise ValueError("distributed_step: coords must be CUDA tensors")
        main = torch.cuda.current_stream(x.device)
        if getattr(self, "_comm", None) is None:
            self._comm = torch.cuda.Stream(device=x.device)
        comm = self._comm
        self.accumulate_head(x, t, batch)
        ev = torch.cuda.Event()
        ev.record(main)
        comm.wait_event(ev)
        with torch.cuda.stream(comm):
            dist.all_reduce(self.mlp.gradient_device(), group=group)
            dist.all_reduce(self.loss_device(), group=group)
        for first, count in bounds:
            if e > b:
                self.accumulate_tables(x, first, count)
            ev = torch.cuda.Event()
            ev.record(main)
            comm.wait_event(ev)
            with torch.cuda.stream(comm):
                dist.all_reduce(gview[first * per_level:(first + count) * per_level], group=group)
                if fview is not None:
                    dist.all_reduce(fview[first * per_level:(first + count) * per_level], group=group)
        main.wait_stream(comm)
        loss = self.loss(batch)
        self.update(table_adam, mlp_adam)
        return loss


def level_ranges(levels: int, chunks: int):
    """[(first, count)] covering 0..levels in at most `chunks` near-equal contiguous ranges."""
    chunks = max(1, min(chunks, levels))
    per = (levels + chunks - 1) // chunks
    return [(f, min(per, levels - f)) for f in range(0, levels, per)]


QUEUE_WINDOW = 256  # queued steps between two loss read-backs in train_field (the ring holds 4096)

BatchSampler = Callable[[int, int], tuple]  # (step, batch) -> (coords [B, dim], targets [B, out_w]) CUDA tensors


def train_field(encoder, mlp, sampler: BatchSampler, cfg: TrainConfig, group=None) -> TrainResult:
    """sxen::train_field (src/trainer.cpp:53-139)."""
    if cfg.batch_size < 1:
        raise ValueError("train: batch_size must be >= 1")
    if cfg.steps < 0:
        raise ValueError("train: steps must be >= 0")
    if cfg.aux_dims < 0:
        raise ValueError("train: aux_dims must be >= 0")
    if cfg.record_every < 1:
        raise ValueError("train: record_every must be >= 1")
    if sampler is None:
        raise ValueError("train: sampler must be callable")
    trainer = Trainer(encoder, mlp, cfg.aux_dims)
    if cfg.reproducible:
        trainer.set_reproducible(True)
    distributed = False
    if group is not None:
        distributed = True
    else:
        try:
            import torch.distributed as dist
            distributed = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
        except Exception:
            distributed = False
    result = TrainResult()

    def record(step: int, loss: float) -> None:
        if not math.isfinite(loss):
            raise TrainingError(f"loss became non-finite at step {step}")
        if step % cfg.record_every == 0 or step == cfg.steps - 1:
            result.loss_curve.append((step, loss))
        result.final_loss = loss

    def draw(step: int):
        """(coords, targets) from the sampler; with aux_dims > 0 it returns (coords, aux, targets) and the aux tensor is
        handed to the trainer for this batch (BatchSampler's three spans, include/sxen/trainer.hpp:26-32)."""
        got = sampler(step, cfg.batch_size)
        if cfg.aux_dims > 0:
            if len(got) != 3:
                raise ValueError("train: with aux_dims > 0 the sampler returns (coords, aux, targets)")
            coords, aux, targets = got
            if aux.shape[0] != coords.shape[0]:
                raise ValueError("train: aux batch size differs from coords")
            trainer.set_aux(aux)
            return coords, targets
        return got[0], got[-1]

    if distributed:
        if cfg.aux_dims > 0:
            raise ValueError("train: aux_dims > 0 is single-GPU on the device path")
        for step in range(cfg.steps):
            coords, targets = draw(step)
            record(step, trainer.distributed_step(coords, targets, cfg.table_adam, cfg.mlp_adam, group))
    else:
        # Single GPU: steps are queued back to back (no host round trip per step) and their losses read in windows;
        # the device gate keeps the reference's "throw before the update" for a non-finite loss.
        first = 0
        keep = []   # aux tensors of the queued steps stay alive until their window is collected
        for step in range(cfg.steps):
            coords, targets = draw(step)
            keep.append(trainer._aux)
            trainer.step_enqueue(coords, targets, cfg.table_adam, cfg.mlp_adam)
            if step + 1 - first == QUEUE_WINDOW or step == cfg.steps - 1:
                losses, _ = trainer.collect()
                for k, loss in enumerate(losses):
                    record(first + k, loss)
                first = step + 1
                keep.clear()
    result.steps_run = cfg.steps
    return result
