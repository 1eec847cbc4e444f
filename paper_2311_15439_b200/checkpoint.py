"""Checkpoint mirror (include/sxen/checkpoint.hpp:17-31, src/checkpoint.cpp:81-175): the reference's little-endian
"SXEN" / "SXML" binary format, so models trained on the B200 load into the reference (and the other way round).

    "SXEN" | version u32 | n, L, T, F, N_base u32 | growth f64 | backend u32 | L blocks of T*F f32
    ["SXML" | version u32 | layer_count, input, hidden, output u32 | per layer: out*in f32 weights, out f32 biases]

Host-side file I/O only; parameters move through HashEncoder.table / Mlp.parameters."""
from __future__ import annotations

import struct
from typing import Optional, Tuple

import numpy as np

from .encoding import Backend, EncoderConfig, HashEncoder, LevelScale
from .errors import IoError
from .mlp import Mlp, MlpConfig

ENCODER_MAGIC, MLP_MAGIC = b"SXEN", b"SXML"
ENCODER_VERSION, MLP_VERSION = 1, 1


def save_checkpoint(path: str, encoder: HashEncoder, mlp: Optional[Mlp] = None) -> None:
    """sxen::save_checkpoint (src/checkpoint.cpp:81-112)."""
    ec = encoder.config
    try:
        with open(path, "wb") as f:
            f.write(ENCODER_MAGIC)
            f.write(struct.pack("<6I", ENCODER_VERSION, ec.dim, ec.levels, ec.table_size, ec.features, ec.base_resolution))
            f.write(struct.pack("<d", float(ec.growth)))
            f.write(struct.pack("<I", 0 if ec.backend == Backend.simplex else 1))
            for l in range(ec.levels):
                f.write(np.ascontiguousarray(encoder.table(l), dtype="<f4").tobytes())
            if mlp is not None:
                mc = mlp.config
                f.write(MLP_MAGIC)
                f.write(struct.pack("<5I", MLP_VERSION, mc.layer_count(), mc.input_width, mc.hidden_width, mc.output_width))
                # parameters() is already "per layer: weights then biases" (src/mlp.cpp:19-32)
                f.write(np.ascontiguousarray(mlp.parameters(), dtype="<f4").tobytes())
    except OSError as exc:
        raise IoError(f"cannot open '{path}' for writing") from exc


def _read(f, n: int) -> bytes:
    b = f.read(n)
    if len(b) != n:
        raise IoError("checkpoint: unexpected end of file")  # src/checkpoint.cpp read_bytes
    return b


def load_checkpoint(path: str, level_scale: int = LevelScale.raw, device: int = 0) -> Tuple[HashEncoder, Optional[Mlp]]:
    """sxen::load_checkpoint (src/checkpoint.cpp:114-175). Returns (encoder, mlp or None)."""
    try:
        f = open(path, "rb")
    except OSError as exc:
        raise IoError(f"cannot open '{path}' for reading") from exc
    with f:
        if _read(f, 4) != ENCODER_MAGIC:
            raise IoError("checkpoint: bad encoder section magic")
        version, dim, levels, table_size, features, base = struct.unpack("<6I", _read(f, 24))
        if version != ENCODER_VERSION:
            raise IoError(f"checkpoint: unsupported encoder section version {version}")
        (growth,) = struct.unpack("<d", _read(f, 8))
        (backend_tag,) = struct.unpack("<I", _read(f, 4))
        if backend_tag > 1:
            raise IoError("checkpoint: unknown backend tag")
        ec = EncoderConfig(dim=dim, levels=levels, table_size=table_size, features=features, base_resolution=base,
                           growth=growth, backend=Backend(backend_tag), level_scale=level_scale)
        try:
            ec.validate()
        except ValueError as exc:
            raise IoError(f"checkpoint: invalid encoder config: {exc}") from exc
        encoder = HashEncoder(ec, device=device)
        per = table_size * features
        for l in range(levels):
            encoder.set_table(l, np.frombuffer(_read(f, 4 * per), dtype="<f4"))
        head = f.read(4)
        if head == b"":
            return encoder, None
        if head != MLP_MAGIC:
            raise IoError("checkpoint: bad mlp section magic")
        mlp_version, layer_count, inp, hid, out = struct.unpack("<5I", _read(f, 20))
        if mlp_version != MLP_VERSION:
            raise IoError(f"checkpoint: unsupported mlp section version {mlp_version}")
        if layer_count < 1:
            raise IoError("checkpoint: mlp layer count must be >= 1")
        mc = MlpConfig(inp, hid, layer_count - 1, out)
        try:
            mc.validate()
        except ValueError as exc:
            raise IoError(f"checkpoint: invalid mlp config: {exc}") from exc
        mlp = Mlp(mc, device=device)
        mlp.set_parameters(np.frombuffer(_read(f, 4 * mlp.parameter_count()), dtype="<f4"))
        if f.read(1) != b"":
            raise IoError("checkpoint: trailing bytes after mlp section")
        return encoder, mlp
