"""Seeded streams and sorted uniforms on the GPU (drop-in for dacresample.randkit).

Mirrors /root/reference/pkg/src/dacresample/randkit.py: ``RngStream``
(:16-62), ``uniform_open`` (:65-67) and ``sorted_uniforms`` (:70-101).

Generator change: the reference's ``RngStream`` is
PCG64 under a SeedSequence; this one is Philox4x64-10 under the same
SeedSequence, in numpy's exact convention (``np.random.Philox``), so that
every GPU thread can jump straight to its own draw.  Same seed => same
sequence across runs; equal in distribution to the reference, not equal
value for value.  ``seed``, ``draws`` and ``substream`` keep their meaning.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._tensors import empty_f64, status_word, to_device_f64

__all__ = ["RngStream", "DeviceRngStream", "uniform_open", "sorted_uniforms"]


class RngStream:
    """Deterministic uniform source with independent substreams (randkit.py:16-62).

    State = (Philox key from ``SeedSequence(seed, spawn_key)``, raw draw
    position).  Single-owner, like the reference.
    """

    __slots__ = ("seed", "draws", "_spawn_key", "_key", "_pos")

    def __init__(self, seed: int, _spawn_key: tuple[int, ...] = ()):
        self.seed = int(seed)
        self._spawn_key = tuple(int(k) for k in _spawn_key)
        seq = np.random.SeedSequence(self.seed, spawn_key=self._spawn_key)
        k = seq.generate_state(2, np.uint64)
        self._key = (int(k[0]), int(k[1]))
        self._pos = 0
        self.draws = 0  # uniform variates served so far

    def substream(self, key: int) -> "RngStream":
        """Independent stream derived from this one; distinct keys never overlap."""
        return RngStream(self.seed, self._spawn_key + (int(key),))

    @property
    def key(self) -> tuple[int, int]:
        return self._key

    @property
    def position(self) -> int:
        """Raw draws consumed so far (the Philox draw offset of the next draw)."""
        return self._pos

    def _take(self, k: int) -> int:
        off = self._pos
        self._pos += k
        self.draws += k
        return off

    def uniforms_device(self, k: int) -> torch.Tensor:
        """k doubles in (0, 1) as a CUDA tensor, advancing the stream."""
        k = int(k)
        if k < 0:
            raise ValueError("negative dimensions are not allowed")
        out = empty_f64(k)
        off = self._take(k)
        if k:
            _lib.check(
                _lib.lib().dr_uniforms(self._key[0], self._key[1], off, k, out.data_ptr(), _lib.stream_handle()),
                "dr_uniforms",
            )
        return out

    def uniform(self) -> float:
        """One double strictly inside (0, 1), advancing the stream."""
        return float(self.uniforms_device(1).item())

    def uniforms(self, k: int) -> np.ndarray:
        """k doubles strictly inside (0, 1) as a float64 array."""
        return self.uniforms_device(k).cpu().numpy()

    def normals(self, shape):
        raise NotImplementedError(
            "RngStream.normals feeds only the weight-field generators (weightgen.py), "
            "which are outside the resampling path this package implements"
        )

    def __repr__(self):
        return f"RngStream(seed={self.seed}, substream={self._spawn_key})"


class DeviceRngStream:
    """An RngStream whose draw position lives in device memory.

    The samplers read the position on the device and advance it there, so a
    sampler call can be captured once in a CUDA graph and replayed with fresh
    draws on every replay (the loop of a particle filter).  Same key
    derivation and draw sequence as :class:`RngStream`; ``position`` reads
    the device counter (synchronising).
    """

    __slots__ = ("seed", "_spawn_key", "_key", "offset_tensor")

    def __init__(self, seed: int, _spawn_key: tuple[int, ...] = (), position: int = 0):
        self.seed = int(seed)
        self._spawn_key = tuple(int(k) for k in _spawn_key)
        k = np.random.SeedSequence(self.seed, spawn_key=self._spawn_key).generate_state(2, np.uint64)
        self._key = (int(k[0]), int(k[1]))
        self.offset_tensor = torch.tensor([int(position)], dtype=torch.int64, device=_lib.device())

    @property
    def key(self) -> tuple[int, int]:
        return self._key

    @property
    def position(self) -> int:
        return int(self.offset_tensor.item())

    @property
    def draws(self) -> int:
        return self.position

    def __repr__(self):
        return f"DeviceRngStream(seed={self.seed}, substream={self._spawn_key})"


def uniform_open(stream: RngStream) -> float:
    """Single uniform draw in the open interval (0, 1) (randkit.py:65-67)."""
    return stream.uniform()


def sorted_uniforms_device(stream, n: int) -> torch.Tensor:
    """:func:`sorted_uniforms` leaving the result on the device (no host sync)."""
    n = int(n)
    if n < 0:
        raise ValueError("n must be >= 0")
    if n == 0:
        return empty_f64(0)
    L = _lib.lib()
    U = empty_f64(n)
    st = status_word()
    ws, wsb = _lib.workspace(L.dr_workspace_bytes(_lib.OP_SORTED, 0, n, 0))
    s = _lib.stream_handle()
    if isinstance(stream, RngStream):
        off = stream._take(n + 1)
        _lib.check(
            L.dr_sorted_uniforms(stream._key[0], stream._key[1], off, n, U.data_ptr(), st.data_ptr(), ws, wsb, s),
            "dr_sorted_uniforms",
        )
    else:
        # duck-typed host stream (e.g. the reference tests' ReplayStream):
        # same kernels, uniforms supplied instead of generated
        raw, _ = to_device_f64(stream.uniforms(n + 1))
        _lib.check(
            L.dr_sorted_uniforms_from(raw.data_ptr(), n, U.data_ptr(), st.data_ptr(), ws, wsb, s),
            "dr_sorted_uniforms_from",
        )
    return U


def sorted_uniforms(stream, n: int) -> np.ndarray:
    """n strictly increasing uniform(0,1) order statistics in O(n) (randkit.py:70-101).

    Draws exactly n + 1 uniforms, maps them to exponential spacings
    z = -log(u), and returns the normalized partial sums Z_i / Z_{n+1},
    repairing the rare float collapse by single-ulp nudges exactly as the
    reference does.
    """
    n = int(n)
    if n < 0:
        raise ValueError("n must be >= 0")
    if n == 0:
        return np.empty(0, dtype=np.float64)
    return sorted_uniforms_device(stream, n).cpu().numpy()
