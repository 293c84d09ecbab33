"""Python mirror of the TC ExecutionEngine over the
tc-b200 C ABI:

    ee = ExecutionEngine()
    ee.define('''def tmm(float(M,K) A, float(N,K) B) -> (C) {
                     C(m,n) +=! A(m,kk) * B(n,kk) }''')
    C = ee.tmm(A, B)          # compile (cache hit / default) and run

Tensors may be CUDA torch tensors (device pointers are passed straight
through, on torch's current stream), CPU torch tensors or numpy arrays (the
library copies in and out; pass pinned memory for fast copies). float32 and
int32 only, dense row-major — the reference's tensor model
(tensor_data.h:23-43).
"""
from __future__ import annotations

import ctypes as C
import json

import numpy as np

from . import _lib
from ._lib import TCB_DEVICE, TCB_F32, TCB_HOST, TCB_I32, TcError, Tensor, check, lib

try:  # torch is plumbing for device memory and streams
    import torch
except Exception:  # pragma: no cover
    torch = None


def _desc(t, shape_only=False) -> Tensor:
    d = Tensor()
    if t is None:
        d.rank = 0
        return d
    if isinstance(t, (tuple, list)):  # a bare shape
        d.rank = len(t)
        for i, e in enumerate(t):
            d.shape[i] = int(e)
        d.dtype = TCB_F32
        return d
    if torch is not None and isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise TcError(23, "tensors must be contiguous (row-major)")
        if t.dtype == torch.float32:
            d.dtype = TCB_F32
        elif t.dtype == torch.int32:
            d.dtype = TCB_I32
        else:
            raise TcError(23, f"unsupported dtype {t.dtype} (float32/int32 only)")
        d.data = t.data_ptr()
        d.location = TCB_DEVICE if t.is_cuda else TCB_HOST
        shape = t.shape
    else:
        a = t
        if not isinstance(a, np.ndarray) or not a.flags.c_contiguous:
            raise TcError(23, "expected a contiguous numpy array or torch tensor")
        if a.dtype == np.float32:
            d.dtype = TCB_F32
        elif a.dtype == np.int32:
            d.dtype = TCB_I32
        else:
            raise TcError(23, f"unsupported dtype {a.dtype} (float32/int32 only)")
        d.data = a.ctypes.data
        d.location = TCB_HOST
        shape = a.shape
    d.rank = len(shape)
    for i, e in enumerate(shape):
        d.shape[i] = int(e)
    return d


def _arr(ts):
    ts = list(ts or [])
    arr = (Tensor * max(1, len(ts)))()
    for i, t in enumerate(ts):
        arr[i] = _desc(t)
    return arr, len(ts)


class ExecutionEngine:
    """define / infer_output_tensor_info / compile / run / tune."""

    def __init__(self, define_builtins: bool = True):
        h = C.c_void_p()
        check(lib.tcb_engine_create(C.byref(h)))
        self._h = h
        self._handles = {}
        if define_builtins:
            self.define(lib.tcb_builtin_ops().decode())

    def __del__(self):
        try:
            lib.tcb_engine_destroy(self._h)
        except Exception:
            pass

    # ------------------------------------------------------------- define
    def define(self, language: str):
        check(lib.tcb_define(self._h, language.encode()))

    def signature(self, name: str):
        np_, nr = C.c_int(), C.c_int()
        b = _lib.buf(4096)
        check(lib.tcb_def_signature(self._h, name.encode(), C.byref(np_), C.byref(nr), b, 4096))
        p, r = b.value.decode().split(";")
        return (p.split(",") if p else []), (r.split(",") if r else [])

    def infer_output_tensor_info(self, name, inputs, outputs=None):
        ins, nin = _arr(inputs)
        _, rets = self.signature(name)
        outs = (Tensor * len(rets))()
        for i, o in enumerate(outputs or []):
            if o is not None:
                outs[i] = _desc(o)
        check(lib.tcb_infer_outputs(self._h, name.encode(), ins, nin, outs, len(rets)))
        return [tuple(outs[i].shape[d] for d in range(outs[i].rank)) for i in range(len(rets))]

    # ------------------------------------------------------------ compile
    def compile(self, name, inputs, outputs=None, options=None, math="ffma") -> int:
        """math: "ffma" (default; FFMA-exact, bit-identical to the reference
        interpreter), "tf32" or "3xtf32" (tcgen05 tensor cores; stated
        tolerance)."""
        ins, nin = _arr(inputs)
        outs, nout = _arr(outputs) if outputs is not None else (None, 0)
        h = C.c_uint64()
        opt = None
        if options is not None:
            opt = (options if isinstance(options, str) else json.dumps(options)).encode()
        if math not in _lib.MATH_MODES:
            raise ValueError(f"math must be one of {sorted(_lib.MATH_MODES)}")
        check(lib.tcb_compile_ex(self._h, name.encode(), ins, nin, outs, nout, opt, _lib.MATH_MODES[math],
                                 C.byref(h)))
        return h.value

    def describe(self, handle: int) -> dict:
        b = _lib.buf(1 << 16)
        check(lib.tcb_describe(self._h, handle, b, 1 << 16))
        return json.loads(b.value.decode())

    # ---------------------------------------------------------------- run
    def run(self, handle, inputs, outputs, stream=None, profile=False, check_errors=True, sync=True):
        """Runs a compiled handle. Returns the device time in ns when profiling.

        sync=False with host tensors only enqueues the copies and the launch
        on `stream` (TCB_RUN_ASYNC); synchronise the stream before reading
        the outputs, then call check() for LUT index errors."""
        ins, nin = _arr(inputs)
        outs, nout = _arr(outputs)
        if stream is None and torch is not None and any(
                isinstance(t, torch.Tensor) and t.is_cuda for t in list(inputs) + list(outputs)):
            stream = torch.cuda.current_stream().cuda_stream
        flags = ((_lib.TCB_RUN_PROFILE if profile else 0) | (0 if check_errors else _lib.TCB_RUN_NOCHECK) |
                 (0 if sync else _lib.TCB_RUN_ASYNC))
        dur = C.c_int64(0)
        check(lib.tcb_run(self._h, handle, ins, nin, outs, nout, C.c_void_p(stream or 0), flags,
                          C.byref(dur)))
        return dur.value if profile else None

    def shard_range(self, handle, rank, world):
        """(lo, hi, extent): rank's balanced slice of the handle's batch
        dimension (tcb_shard_range)."""
        lo, hi, n = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.tcb_shard_range(self._h, handle, rank, world, C.byref(lo), C.byref(hi), C.byref(n)))
        return lo.value, hi.value, n.value

    def run_shard(self, handle, inputs, outputs, rank, world, stream=None, check_errors=True):
        """Runs only this rank's batch slice of a handle compiled for the
        full shapes, in place on the full device tensors (tcb_run_shard)."""
        ins, nin = _arr(inputs)
        outs, nout = _arr(outputs)
        if stream is None and torch is not None:
            stream = torch.cuda.current_stream().cuda_stream
        flags = 0 if check_errors else _lib.TCB_RUN_NOCHECK
        check(lib.tcb_run_shard(self._h, handle, ins, nin, outs, nout, rank, world, C.c_void_p(stream or 0),
                                flags))

    def check(self, handle):
        check(lib.tcb_check(self._h, handle))

    def release(self, handle):
        """Frees a compiled handle's device staging and error flag
        (tcb_release); the handle must not be used afterwards."""
        check(lib.tcb_release(self._h, handle))

    def prepare(self, handle, inputs, outputs) -> "PreparedRun":
        """Binds tensors to a compiled handle once, like the reference's
        caller building its DLTensor arrays once (execution_engine.h:93-101);
        PreparedRun.run() then only crosses the C ABI."""
        return PreparedRun(self, handle, inputs, outputs)

    # --------------------------------------------------------------- tune
    def tune(self, name, inputs, outputs=None, **opts) -> dict:
        ins, nin = _arr(inputs)
        outs, nout = _arr(outputs) if outputs is not None else (None, 0)
        b = _lib.buf(1 << 14)
        check(lib.tcb_tune(self._h, name.encode(), ins, nin, outs, nout, json.dumps(opts).encode(), b,
                           1 << 14))
        return json.loads(b.value.decode())

    def default_options(self, name, inputs, outputs=None) -> dict:
        ins, nin = _arr(inputs)
        outs, nout = _arr(outputs) if outputs is not None else (None, 0)
        b = _lib.buf(4096)
        check(lib.tcb_options_default(self._h, name.encode(), ins, nin, outs, nout, b, 4096))
        return json.loads(b.value.decode())

    def canonical(self, name, inputs, outputs=None):
        ins, nin = _arr(inputs)
        outs, nout = _arr(outputs) if outputs is not None else (None, 0)
        c, k = _lib.buf(1 << 16), _lib.buf(1 << 16)
        check(lib.tcb_canonical(self._h, name.encode(), ins, nin, outs, nout, c, 1 << 16, k, 1 << 16))
        return c.value.decode(), k.value.decode()

    def cache_lookup(self, name, inputs, outputs=None):
        ins, nin = _arr(inputs)
        outs, nout = _arr(outputs) if outputs is not None else (None, 0)
        hit = C.c_int(0)
        b = _lib.buf(4096)
        check(lib.tcb_cache_lookup(self._h, name.encode(), ins, nin, outs, nout, C.byref(hit), b, 4096))
        return json.loads(b.value.decode()) if hit.value else None

    def cache_inject(self, name, inputs, options, cost, outputs=None):
        ins, nin = _arr(inputs)
        outs, nout = _arr(outputs) if outputs is not None else (None, 0)
        opt = options if isinstance(options, str) else json.dumps(options)
        check(lib.tcb_cache_inject(self._h, name.encode(), ins, nin, outs, nout, opt.encode(), cost))

    def session_inputs(self, name, shapes, seed, outputs=None):
        """tuner::makeSessionInputs: host numpy tensors for every parameter."""
        params, _ = self.signature(name)
        arrays = []
        for s in shapes:
            arrays.append(np.empty(s, np.float32))
        return self._session_fill(name, arrays, seed, outputs)

    def _session_fill(self, name, arrays, seed, outputs=None):
        ins, nin = _arr(arrays)
        outs, nout = _arr(outputs) if outputs is not None else (None, 0)
        check(lib.tcb_session_inputs(self._h, name.encode(), ins, nin, outs, nout, seed))
        return arrays

    # ---------------------------------------------- paper-style ee.name(...)
    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        try:
            self.signature(name)
        except TcError as e:
            raise AttributeError(name) from e

        def call(*inputs, outputs=None, options=None):
            key = (name, tuple(tuple(t.shape) for t in inputs),
                   json.dumps(options, sort_keys=True) if options else None)
            if outputs is None:
                shapes = self.infer_output_tensor_info(name, inputs)
                dev = inputs[0].device if torch is not None and isinstance(inputs[0], torch.Tensor) else None
                if dev is not None:
                    outputs = [torch.zeros(s, dtype=torch.float32, device=dev) for s in shapes]
                else:
                    outputs = [np.zeros(s, np.float32) for s in shapes]
            h = self._handles.get(key)
            if h is None:
                h = self._handles[key] = self.compile(name, inputs, outputs, options)
            self.run(h, inputs, outputs)
            return outputs[0] if len(outputs) == 1 else tuple(outputs)

        return call


def tensor_file_write(path, array):
    """Writes a numpy float32/int32 array as a TCTN1 file (the reference's
    writeTensorFile format, tensor_data.cc:122-147)."""
    a = np.ascontiguousarray(array)
    if a.dtype not in (np.float32, np.int32):
        raise TypeError("TCTN1 tensors are float32 or int32")
    check(lib.tcb_tensor_file_write(str(path).encode(), C.byref(_desc(a))))


def tensor_file_read(path):
    """Reads a TCTN1 file into a numpy array (readTensorFile, tensor_data.cc:149-189)."""
    t = Tensor()
    check(lib.tcb_tensor_file_read(str(path).encode(), C.byref(t)))
    try:
        shape = tuple(t.shape[d] for d in range(t.rank))
        n = int(np.prod(shape)) if shape else 1
        dt = np.int32 if t.dtype == TCB_I32 else np.float32
        buf = (C.c_uint8 * (4 * n)).from_address(t.data)
        return np.frombuffer(bytes(buf), dtype=dt).reshape(shape).copy()
    finally:
        lib.tcb_tensor_file_free(t.data)


def cache_entries():
    """Every cache entry (cache list / inspect)."""
    b = _lib.buf(1 << 24)
    check(lib.tcb_cache_entries(b, 1 << 24))
    return json.loads(b.value.decode())


def cache_load(path):
    check(lib.tcb_cache_load(path.encode()))


def cache_save(path):
    check(lib.tcb_cache_save(path.encode()))


def cache_size():
    return lib.tcb_cache_size()


def cache_purge():
    check(lib.tcb_cache_purge())


def cache_set_history(path):
    check(lib.tcb_cache_set_history(path.encode() if path else b""))


def cache_serialize():
    b = _lib.buf(1 << 22)
    check(lib.tcb_cache_serialize(b, 1 << 22))
    return b.value.decode()


def cache_deserialize(text):
    check(lib.tcb_cache_deserialize(text.encode()))


def fill_uniform(n, seed, lo=-1.0, hi=1.0, dtype=np.float32):
    a = np.empty(n, dtype)
    check(lib.tcb_fill_uniform(a.ctypes.data, n, TCB_I32 if dtype == np.int32 else TCB_F32, seed, lo,
                               hi))
    return a


def options_baseline(i):
    b = _lib.buf(4096)
    check(lib.tcb_options_baseline(i, b, 4096))
    return b.value.decode()


def options_normalize(text):
    b = _lib.buf(4096)
    check(lib.tcb_options_normalize(text.encode(), b, 4096))
    return b.value.decode()


def options_digest(text):
    b = _lib.buf(64)
    check(lib.tcb_options_digest(text.encode(), b, 64))
    return b.value.decode()


def options_validate(text):
    check(lib.tcb_options_validate(text.encode()))


def version():
    return lib.tcb_version().decode()


def measure_peaks(dev=0):
    """Device peaks not in MEASURED_PEAKS.json (fp32 FFMA TFLOP/s), measured now."""
    import json
    b = _lib.buf(1024)
    check(lib.tcb_measure_peaks(dev, b, 1024))
    return json.loads(b.value.decode())


def device_info(dev=0):
    b = _lib.buf(1024)
    check(lib.tcb_device_info(dev, b, 1024))
    return b.value.decode()


class PreparedRun:
    """A handle bound to fixed tensors (their descriptors are built once).
    The tensors are kept alive; writing new values into them between runs is
    the intended use."""

    def __init__(self, ee, handle, inputs, outputs):
        self.ee, self.handle = ee, handle
        self.tensors = (list(inputs), list(outputs))
        self._ins, self._nin = _arr(inputs)
        self._outs, self._nout = _arr(outputs)
        self._cuda = torch is not None and any(isinstance(t, torch.Tensor) and t.is_cuda
                                               for t in self.tensors[0] + self.tensors[1])

    def run(self, stream=None, sync=True, check_errors=True):
        """One call; see ExecutionEngine.run for `sync`."""
        if stream is None and self._cuda:
            stream = torch.cuda.current_stream().cuda_stream
        flags = (0 if check_errors else _lib.TCB_RUN_NOCHECK) | (0 if sync else _lib.TCB_RUN_ASYNC)
        check(lib.tcb_run(self.ee._h, self.handle, self._ins, self._nin, self._outs, self._nout,
                          C.c_void_p(stream or 0), flags, None))
