"""On-disk formats of the reference detector, ingested straight into the
device path:

* NOMA1 binary transmission dataset (io.hpp:10-19, io.cpp:80-136): magic
  "NOMA1", u16 version 1, u32 K, M, N_T, N_D, then f64 powers[K], the channel
  (M x K), X_T (N_T x M), Y_T (N_T x K), X_D (N_D x M), Y_D (N_D x K) as
  row-major interleaved complex f64, and a trailing f64 noise power
  (io.cpp:96/:122 -- the header comment omits it).  Little-endian, packed:
  every f64 after the 23-byte header sits at an odd offset, so the arrays
  are copied into aligned buffers; their row-major [t][m] order already is
  the device layout (`to_device_slot`).
* noma-net detector parameters (io.cpp:138-211): a JSON document
  {"format": "noma-net", "version": 1, "user_index", "config_digest", "dims",
  "w0", "layers": [{"weights": rows, "bias"}], "final_weights"}; nlohmann's
  dump() sorts object keys and writes compact separators with shortest
  round-trip numbers, which json.dumps(sort_keys=True, separators=(",", ":"))
  reproduces.

Errors follow errors.hpp:23-35: IoError (cannot open / write), FormatError
(bad magic, version, zero dimension, malformed params) and TruncationError
(length inconsistent with the header).
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

MAGIC = b"NOMA1"
VERSION = 1
_HDR = struct.Struct("<5sHIIII")  # 23 bytes


class IoError(OSError):
    """noma::io_error"""


class FormatError(IoError):
    """noma::format_error"""


class TruncationError(IoError):
    """noma::truncation_error"""


@dataclass
class TransmissionRecord:
    """TransmissionRecord (channel_sim.hpp:52-61)."""
    channel: np.ndarray        # M x K complex128
    powers: np.ndarray         # K
    train_rx: np.ndarray       # N_T x M
    train_symbols: np.ndarray  # N_T x K
    data_rx: np.ndarray        # N_D x M
    data_symbols: np.ndarray   # N_D x K
    noise_power: float


def write_dataset(rec: TransmissionRecord, path: str) -> None:
    """write_dataset (io.cpp:80-97)."""
    M, K = rec.channel.shape
    parts = [_HDR.pack(MAGIC, VERSION, K, M, rec.train_rx.shape[0], rec.data_rx.shape[0]),
             np.ascontiguousarray(rec.powers, dtype="<f8").tobytes()]
    for a in (rec.channel, rec.train_rx, rec.train_symbols, rec.data_rx, rec.data_symbols):
        parts.append(np.ascontiguousarray(a, dtype="<c16").tobytes())
    parts.append(struct.pack("<d", rec.noise_power))
    try:
        with open(path, "wb") as f:
            f.write(b"".join(parts))
    except OSError as e:
        raise IoError(f"cannot open for writing: {path}") from e


def read_dataset(path: str) -> TransmissionRecord:
    """read_dataset (io.cpp:99-136), same checks in the same order."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError(f"cannot open for reading: {path}") from e
    if len(data) < 5:
        raise TruncationError("file shorter than its header promises")
    if data[:5] != MAGIC:
        raise FormatError(f"bad magic; not a NOMA1 dataset: {path}")
    if len(data) < 7:
        raise TruncationError("file shorter than its header promises")
    if struct.unpack_from("<H", data, 5)[0] != VERSION:
        raise FormatError("unsupported dataset version")
    if len(data) < _HDR.size:
        raise TruncationError("file shorter than its header promises")
    _, _, K, M, NT, ND = _HDR.unpack_from(data, 0)
    if 0 in (K, M, NT, ND):
        raise FormatError("zero dimension in dataset header")
    expected = _HDR.size + 8 * K + 16 * (M * K + NT * M + NT * K + ND * M + ND * K) + 8
    if len(data) != expected:
        raise TruncationError("dataset length inconsistent with header dims")
    off = _HDR.size

    def take(shape, dtype):
        nonlocal off
        n = int(np.prod(shape)) * np.dtype(dtype).itemsize
        # np.frombuffer on the unaligned slice, then an aligned copy
        a = np.frombuffer(data, dtype=dtype, count=int(np.prod(shape)), offset=off).reshape(shape).copy()
        off += n
        return a

    powers = take((K,), "<f8").astype(np.float64)
    ch = take((M, K), "<c16").astype(np.complex128)
    trx = take((NT, M), "<c16").astype(np.complex128)
    tsy = take((NT, K), "<c16").astype(np.complex128)
    drx = take((ND, M), "<c16").astype(np.complex128)
    dsy = take((ND, K), "<c16").astype(np.complex128)
    noise = struct.unpack_from("<d", data, off)[0]
    return TransmissionRecord(ch, powers, trx, tsy, drx, dsy, noise)


def to_device_slot(rec: TransmissionRecord):
    """One slot of device inputs for noma_pipeline: pilot_rx [1][N_T][M] c64,
    pilot_sym [1][N_T][K] c64, data_rx [1][N_D][M] c32 (the FP32 data phase)
    and truth codes [1][N_D][K] (hard_decision_qpsk of Y_D, eval.cpp:38-45)."""
    from .api import codes_of

    return (rec.train_rx[None], rec.train_symbols[None],
            rec.data_rx.astype(np.complex64)[None], codes_of(rec.data_symbols)[None])


# ------------------------------------------------------------- noma-net
@dataclass
class LoadedParams:
    """LoadedParams (io.hpp:28-32) over the reference's parameter set."""
    dims: List[int]
    w0: np.ndarray
    layers: List[tuple]          # (W_n [L_n x L_{n-1}], b_n [L_n])
    final_weights: np.ndarray
    user_index: int = 0
    config_digest: str = ""


def write_params(dims, w0, layers, final_weights, user_index: int, config_digest: str, path: str) -> None:
    """write_params (io.cpp:138-168)."""
    doc = {
        "format": "noma-net", "version": 1, "user_index": int(user_index),
        "config_digest": config_digest, "dims": [int(d) for d in dims],
        "w0": [float(v) for v in np.asarray(w0).ravel()],
        "layers": [{"weights": [[float(v) for v in row] for row in np.asarray(W)],
                    "bias": [float(v) for v in np.asarray(b).ravel()]} for W, b in layers],
        "final_weights": [float(v) for v in np.asarray(final_weights).ravel()],
    }
    try:
        with open(path, "w") as f:
            f.write(json.dumps(doc, sort_keys=True, separators=(",", ":")))
    except OSError as e:
        raise IoError(f"cannot open for writing: {path}") from e


def read_params(path: str) -> LoadedParams:
    """read_params (io.cpp:170-211)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError as e:
        raise IoError(f"cannot open params file: {path}") from e
    try:
        doc = json.loads(text)
    except json.JSONDecodeError as e:
        raise FormatError(f"bad params file: {e}") from e
    if not isinstance(doc, dict) or doc.get("format") != "noma-net":
        raise FormatError(f"not a noma-net params file: {path}")
    try:
        layers = []
        for layer in doc["layers"]:
            rows = layer["weights"]
            width = len(rows[0]) if rows else 0
            if any(len(r) != width for r in rows):
                raise FormatError("ragged weight matrix in params file")
            layers.append((np.array(rows, dtype=np.float64).reshape(len(rows), width),
                           np.array(layer["bias"], dtype=np.float64)))
        return LoadedParams([int(d) for d in doc["dims"]], np.array(doc["w0"], dtype=np.float64),
                            layers, np.array(doc["final_weights"], dtype=np.float64),
                            int(doc["user_index"]), str(doc.get("config_digest", "")))
    except (KeyError, TypeError, ValueError) as e:
        raise FormatError(f"bad params file: {e}") from e
