"""Device-side field vectors (torch tensors as plain memory) and scalar codecs.

A field vector of n elements is a torch.int64 CUDA tensor of shape (n, W),
W = 4 (BLS12-381 Fr, 32-byte Montgomery limbs) or 1 (2^61-1, canonical).
Torch is only the allocator / stream provider here; all arithmetic runs in
libzkl_b200.so.
"""

import ctypes

import numpy as np
import torch

from . import _native as N

MODULUS = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001
TEST_MODULUS = (1 << 61) - 1


class UnsupportedField(ValueError):
    """The GPU backend implements the reference's two prover fields only."""


class FieldSpec:
    __slots__ = ("modulus", "fid", "nbytes", "words")

    def __init__(self, modulus, fid, nbytes):
        self.modulus = modulus
        self.fid = fid
        self.nbytes = nbytes
        self.words = nbytes // 8


FR = FieldSpec(MODULUS, 0, 32)
M61 = FieldSpec(TEST_MODULUS, 1, 8)


def spec_for(modulus):
    """Field spec for a reference modulus; requires the CUDA backend."""
    if modulus == MODULUS:
        spec = FR
    elif modulus == TEST_MODULUS:
        spec = M61
    else:
        raise UnsupportedField("no GPU field for modulus %d" % modulus)
    N.lib()  # raises BackendUnavailable: no CPU fallback
    return spec


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def empty(spec, n):
    return torch.empty((max(n, 1), spec.words), dtype=torch.int64, device="cuda")


def scalar_bytes(v, spec):
    return (int(v) % spec.modulus).to_bytes(spec.nbytes, "little")


def scalars_bytes(vals, spec):
    p, nb = spec.modulus, spec.nbytes
    return b"".join((int(v) % p).to_bytes(nb, "little") for v in vals)


def encode(values, spec):
    """Python ints -> canonical little-endian bytes (reduced mod p)."""
    p = spec.modulus
    if spec.words == 1:
        arr = np.fromiter((int(v) % p for v in values), dtype=np.uint64, count=len(values))
        return arr.tobytes()
    return b"".join((int(v) % p).to_bytes(32, "little") for v in values)


def upload(values, spec, out=None):
    """Python ints -> device storage form (Montgomery for Fr)."""
    n = len(values)
    host = torch.frombuffer(bytearray(encode(values, spec)), dtype=torch.int64)
    if out is None:
        out = empty(spec, n)
    if n:
        out.view(-1)[: n * spec.words].copy_(host, non_blocking=False)
        N.check(N.lib().zkl_to_mont(spec.fid, ptr(out), ptr(out), n, stream()))
    return out


def decode(raw, spec, n, _fb=int.from_bytes):
    if spec.words == 1:
        return np.frombuffer(raw, dtype=np.uint64, count=n).tolist()
    raw = bytes(raw)
    return [_fb(raw[i:i + 32], "little") for i in range(0, 32 * n, 32)]


def download(buf, spec, n):
    """Device storage -> canonical Python ints."""
    if n == 0:
        return []
    raw = (ctypes.c_uint8 * (n * spec.nbytes))()
    N.check(N.lib().zkl_read(spec.fid, raw, ptr(buf), n, stream()))
    return decode(bytes(raw), spec, n)


def read_scalar(buf, spec, index=0):
    raw = (ctypes.c_uint8 * spec.nbytes)()
    src = ctypes.c_void_p(buf.data_ptr() + index * spec.nbytes)
    N.check(N.lib().zkl_read(spec.fid, raw, src, 1, stream()))
    return int.from_bytes(bytes(raw), "little")


def lift(int_tensor, spec, out=None):
    """Signed int16/int32/int64 CUDA tensor -> field vector (negatives p-|x|)."""
    t = int_tensor.contiguous()
    mt = {torch.int16: N.MT_I16, torch.int32: N.MT_I32, torch.int64: N.MT_I64}[t.dtype]
    n = t.numel()
    if out is None:
        out = empty(spec, n)
    N.check(N.lib().zkl_lift(spec.fid, mt, ptr(out), ptr(t), n, stream()))
    return out


def eq_table(point, spec, out=None):
    m = len(point)
    if out is None:
        out = empty(spec, 1 << m)
    N.check(N.lib().zkl_eq_table(spec.fid, ptr(out), scalars_bytes(point, spec), m, stream()))
    return out


def dot(a, b, spec, n):
    raw = (ctypes.c_uint8 * spec.nbytes)()
    N.check(N.lib().zkl_dot(spec.fid, raw, ptr(a), ptr(b) if b is not None else None, n,
                            stream()))
    return int.from_bytes(bytes(raw), "little")


class DeviceVector:
    """n field elements resident on the GPU (storage form).

    Accepted wherever the reference passes a tuple of field residues
    (SecretVector / LookupTable entries, multiplicity vectors), so large
    lookups never round-trip through Python ints.
    """

    __slots__ = ("buf", "n", "spec")

    def __init__(self, buf, n, spec):
        self.buf, self.n, self.spec = buf, n, spec

    def __len__(self):
        return self.n

    def to_list(self):
        return download(self.buf, self.spec, self.n)


class LiftedColumn(DeviceVector):
    """A DeviceVector backed by a signed integer device column (x mod p):
    the 32-byte field buffer is lifted only when something reads it.  Range
    lookups bin and gather straight from the integers (lookup.py), so their
    secrets are usually never lifted."""

    __slots__ = ("col", "_buf")

    def __init__(self, col, spec):
        self.col = col.reshape(-1)
        self._buf = None
        self.n, self.spec = self.col.numel(), spec

    @property
    def buf(self):
        if self._buf is None:
            self._buf = lift(self.col, self.spec)
        return self._buf

    def value(self, i):
        """Entry i as a canonical residue, without lifting the column."""
        return int(self.col[i]) % self.spec.modulus


class PairColumn(DeviceVector):
    """x + alpha*y over signed integer device columns (a pair lookup's
    compressed secret, tables.py:131-140) as a DeviceVector whose 32-byte field
    buffer is built only when something reads it: pair multiplicities bin from
    the integers and the indexed logUp reads the table side, so for an
    in-table secret the buffer is never written."""

    __slots__ = ("x", "y", "alpha", "_buf")

    def __init__(self, x, y, alpha, spec):
        self.x, self.y = x.contiguous().view(-1), y.contiguous().view(-1)
        self.alpha, self.spec = alpha, spec
        self.n = self.x.numel()
        self._buf = None

    @property
    def buf(self):
        if self._buf is None:
            self._buf = pair_combine(self.x, self.y, self.alpha, self.spec).buf
        return self._buf

    @property
    def materialized(self):
        return self._buf is not None

    def value(self, i):
        p = self.spec.modulus
        return (int(self.x[i]) + self.alpha * int(self.y[i])) % p


def field_buffer(values, spec):
    """Device storage for a DeviceVector or a sequence of residues."""
    if isinstance(values, DeviceVector):
        return values.buf
    return upload(list(values), spec)


def as_list(values):
    return values.to_list() if isinstance(values, DeviceVector) else list(values)


_INT_TYPES = {torch.int16: N.MT_I16, torch.int32: N.MT_I32, torch.int64: N.MT_I64}


IGEMM_LIB = True  # large products through the library int8 GEMM (tests flip it)


def _lib_gemm_shape(M, K, N):
    # torch._int_mm (cuBLASLt int8, tcgen05 on B200) wants K, N multiples of 8
    # and M > 16; the int32 plane products stay exact for K <= 2^16 (|sum| <=
    # 2^14 K).  The planes, four GEMMs and the int64 recombination cost ~0.1 ms
    # of fixed work, so only products of >= 2^32 MACs take this path (the
    # per-head attention products stay on the kernel: 28 us vs 134 us)
    return (M >= 128 and N >= 128 and K % 8 == 0 and N % 8 == 0 and 16 <= K <= (1 << 16)
            and M * K * N >= (1 << 32))


def _igemm16_lib(a, b, c):
    """a @ b from four int8 plane products: hi = a >> 8, lo = (a & 255) - 128,
    so a = 256 hi + lo + 128 and the int64 product is recombined exactly
    (zkl_split_i16 / zkl_igemm_combine around torch._int_mm)."""
    M, K = a.shape
    Nn = b.shape[1]
    ah = torch.empty((M, K), dtype=torch.int8, device=a.device)
    al = torch.empty_like(ah)
    bh = torch.empty((K, Nn), dtype=torch.int8, device=a.device)
    bl = torch.empty_like(bh)
    lib, st = N.lib(), stream()
    N.check(lib.zkl_split_i16(ptr(a), M * K, ptr(ah), ptr(al), st))
    N.check(lib.zkl_split_i16(ptr(b), K * Nn, ptr(bh), ptr(bl), st))
    hh = torch._int_mm(ah, bh)
    hl = torch._int_mm(ah, bl)
    lh = torch._int_mm(al, bh)
    ll = torch._int_mm(al, bl)
    row = a.sum(1, dtype=torch.int64)
    col = b.sum(0, dtype=torch.int64)
    N.check(lib.zkl_igemm_combine(ptr(hh), ptr(hl), ptr(lh), ptr(ll), ptr(row), ptr(col), K,
                                  ptr(c), M, Nn, st))
    return c


def igemm16(a, b, out=None):
    """Exact int64 a @ b for int16 CUDA matrices; `out` an optional
    preallocated contiguous int64 result.  Large products go through the
    library int8 GEMM on byte planes (_igemm16_lib), the rest through the
    repo's byte-sliced mma.sync kernel (zkl_igemm_i16, split-K when skinny)."""
    a, b = a.contiguous(), b.contiguous()
    if a.dtype != torch.int16 or b.dtype != torch.int16 or a.dim() != 2 or b.dim() != 2:
        raise TypeError("igemm16 takes two int16 matrices")
    M, K = a.shape
    K2, Nn = b.shape
    if K != K2:
        raise ValueError("igemm16: inner dimensions %d and %d differ" % (K, K2))
    if out is None:
        c = torch.empty((M, Nn), dtype=torch.int64, device=a.device)
    else:
        if out.shape != (M, Nn) or out.dtype != torch.int64 or not out.is_contiguous():
            raise ValueError("igemm16: out must be a contiguous %dx%d int64 tensor" % (M, Nn))
        c = out
    if M and Nn:
        if IGEMM_LIB and _lib_gemm_shape(M, K, Nn):
            return _igemm16_lib(a, b, c)
        N.check(N.lib().zkl_igemm_i16(ptr(a), ptr(b), ptr(c), M, K, Nn, stream()))
    return c


def pair_combine(x, y, alpha, spec):
    """x + alpha * y for signed integer CUDA tensors (tables.py:131-140)."""
    x = x.contiguous().view(-1)
    y = y.contiguous().view(-1)
    n = x.numel()
    out = empty(spec, n)
    N.check(N.lib().zkl_pair_combine(spec.fid, ptr(out), ptr(x), _INT_TYPES[x.dtype], ptr(y),
                                     _INT_TYPES[y.dtype], n, scalar_bytes(alpha, spec),
                                     stream()))
    return DeviceVector(out, n, spec)


class Staged:
    """Host -> device staging on a copy stream: `stage(host_tensors)` queues
    the copies (pinned host memory: truly asynchronous on the copy engine)
    and returns the device tensors; `ready(i)` makes the current stream wait
    for item i only.  A caller proving a batch of claims stages them all up
    front and proves claim i as soon as its own operands have landed, so the
    PCIe transfer of claim i+1 overlaps the proof of claim i."""

    def __init__(self):
        import torch

        self.torch = torch
        self.copy = torch.cuda.Stream()

    def stage(self, groups, out=None):
        """groups: list of tuples of pinned host tensors -> list of tuples of
        device tensors (reusing `out`'s buffers when given)."""
        torch = self.torch
        start = torch.cuda.Event()
        start.record(torch.cuda.current_stream())
        self.events = []
        dev = []
        with torch.cuda.stream(self.copy):
            self.copy.wait_event(start)  # after the caller's earlier work
            for g, grp in enumerate(groups):
                bufs = out[g] if out is not None else tuple(
                    torch.empty_like(h, device="cuda") for h in grp)
                for d, h in zip(bufs, grp):
                    d.copy_(h, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.copy)
                self.events.append(ev)
                dev.append(bufs)
        return dev

    def ready(self, i):
        self.torch.cuda.current_stream().wait_event(self.events[i])

