"""Test-side ctypes bindings for the oracle (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  — oracle/liboracle.so, the C restatement of the reference
  interpreter's arithmetic (oracle/oracle.c).
* ``RefLib``  — oracle/_ref/libtcref.so, the unmodified reference library
  compiled from /root/reference (oracle/Makefile) behind a C shim
  (oracle/ref_runner.cc). Present in this container and, once built, on
  the GPU box (the .so travels with the snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs use
this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libtcref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
I64 = C.c_int64


def build_oracle():
    if not os.path.exists(ORACLE_SO):
        subprocess.check_call(["make", "-s", "-C", ORACLE_DIR])


class Oracle:
    _lib = None

    def __init__(self):
        if Oracle._lib is None:
            build_oracle()
            lib = C.CDLL(ORACLE_SO)
            lib.orc_rng_new.restype = C.c_void_p
            lib.orc_rng_new.argtypes = [C.c_uint64]
            lib.orc_rng_free.argtypes = [C.c_void_p]
            lib.orc_rng_next.restype = C.c_uint64
            lib.orc_rng_next.argtypes = [C.c_void_p]
            lib.orc_rng_fill_f32.argtypes = [C.c_void_p, _f32p, I64, C.c_double, C.c_double]
            lib.orc_rng_fill_i32.argtypes = [C.c_void_p, _i32p, I64, C.c_double, C.c_double]
            lib.orc_fnv1a64.restype = C.c_uint64
            lib.orc_fnv1a64.argtypes = [C.c_void_p, I64]
            lib.orc_tbmm.argtypes = [_f32p, _f32p, _f32p, I64, I64, I64, I64, C.c_int]
            lib.orc_fc_relu.argtypes = [_f32p, I64, _f32p, I64, _f32p, _f32p, I64, I64, I64]
            lib.orc_kru3.argtypes = [_f32p] * 7 + [I64] * 7
            lib.orc_gconv.argtypes = [_f32p] * 4 + [I64] * 9
            lib.orc_gconv_points.argtypes = [_f32p, _f32p, _f32p, _i64p, I64, _f32p] + [I64] * 9
            lib.orc_lut.restype = C.c_int
            lib.orc_lut.argtypes = [_f32p, I64, I64, _i32p, I64, I64, _f32p]
            lib.orc_set_threads.argtypes = [C.c_int]
            lib.orc_max_threads.restype = C.c_int
            Oracle._lib = lib
        self.lib = Oracle._lib

    # -- deterministic inputs (std::mt19937_64 + libstdc++ distributions) --
    def rng(self, seed):
        return _Rng(self.lib, seed)

    def fnv(self, arr):
        a = np.ascontiguousarray(arr)
        return int(self.lib.orc_fnv1a64(a.ctypes.data, a.nbytes))

    # -- operators --
    def tbmm(self, X, Y, Zin=None):
        B, N, M = X.shape
        K = Y.shape[1]
        Z = np.zeros((B, N, K), np.float32) if Zin is None else np.array(Zin, np.float32, copy=True)
        self.lib.orc_tbmm(X, Y, Z, B, N, M, K, 0 if Zin is None else 1)
        return Z

    def tmm(self, A, Bm):
        return self.tbmm(A[None], Bm[None])[0]

    def c3(self, I3, W, C3in):
        return self.tbmm(I3[None], W[None], C3in[None])[0]

    def fc_relu(self, I, W, bias, kred=None):
        B, ldi = I.shape
        nout, ldw = W.shape
        kred = min(ldi, ldw) if kred is None else kred
        O = np.empty((B, nout), np.float32)
        self.lib.orc_fc_relu(np.ascontiguousarray(I), ldi, np.ascontiguousarray(W), ldw,
                             np.ascontiguousarray(bias), O, B, nout, kred)
        return O

    def mlp3(self, O1, W2, B2, W3, B3, W4, B4):
        O2 = self.fc_relu(O1, W2, B2)
        O3 = self.fc_relu(O2, W3, B3)
        O4 = self.fc_relu(O3, W4, B4)
        return O2, O3, O4

    def kru3(self, W0, W1, W2, X):
        M, N0, N1, N2 = X.shape
        D0, D1, D2 = W0.shape[0], W1.shape[0], W2.shape[0]
        Y = np.empty((M, D0, D1, D2), np.float32)
        XW1 = np.empty((M, N0, D1, D2), np.float32)
        XW2 = np.empty((M, N0, N1, D2), np.float32)
        self.lib.orc_kru3(W0, W1, W2, X, Y, XW1, XW2, M, N0, N1, N2, D0, D1, D2)
        return Y, XW1, XW2

    def gconv(self, I, W1, Bv):
        N, G, Cc, H, W = I.shape
        F, KH, KW = W1.shape[1], W1.shape[3], W1.shape[4]
        O = np.empty((N, G, F, H - KH + 1, W - KW + 1), np.float32)
        self.lib.orc_gconv(I, W1, Bv, O, N, G, Cc, H, W, F, KH, KW, Bv.shape[0])
        return O

    def gconv_points(self, I, W1, Bv, idx):
        N, G, Cc, H, W = I.shape
        F, KH, KW = W1.shape[1], W1.shape[3], W1.shape[4]
        idx = np.ascontiguousarray(idx, np.int64)
        out = np.empty(idx.shape[0], np.float32)
        self.lib.orc_gconv_points(I, W1, Bv, idx, idx.shape[0], out, N, G, Cc, H, W, F, KH, KW,
                                  Bv.shape[0])
        return out

    def lut(self, LUT, I):
        E, D = LUT.shape
        B, L = I.shape
        O = np.empty((B, D), np.float32)
        rc = self.lib.orc_lut(LUT, E, D, np.ascontiguousarray(I, np.int32), B, L, O)
        if rc != 0:
            raise IndexError("IndexOutOfRange")
        return O


class _Rng:
    def __init__(self, lib, seed):
        self.lib = lib
        self.h = lib.orc_rng_new(seed)

    def __del__(self):
        try:
            self.lib.orc_rng_free(self.h)
        except Exception:
            pass

    def next(self):
        return int(self.lib.orc_rng_next(self.h))

    def f32(self, shape, lo=-1.0, hi=1.0):
        a = np.empty(shape, np.float32)
        self.lib.orc_rng_fill_f32(self.h, a.reshape(-1), a.size, lo, hi)
        return a

    def i32(self, shape, lo, hi):
        a = np.empty(shape, np.int32)
        self.lib.orc_rng_fill_i32(self.h, a.reshape(-1), a.size, lo, hi)
        return a


class RefLib:
    """The reference library itself (oracle/_ref/libtcref.so)."""
    _lib = None

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self):
        if RefLib._lib is None:
            lib = C.CDLL(REF_SO)
            cpp = C.POINTER(C.c_char_p)
            lib.tcref_run.restype = C.c_int
            lib.tcref_run.argtypes = [C.c_char_p, C.c_char_p, C.c_int, cpp, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), C.POINTER(I64), C.POINTER(C.c_void_p),
                                      C.c_int, cpp, C.POINTER(C.c_void_p), C.POINTER(I64),
                                      C.POINTER(I64), C.POINTER(C.c_int), C.c_char_p, C.c_int]
            lib.tcref_key.restype = C.c_int
            lib.tcref_key.argtypes = [C.c_char_p, C.c_char_p, C.c_int, cpp, C.POINTER(C.c_int),
                                      C.POINTER(I64), C.c_char_p, C.c_int, C.c_char_p, C.c_int,
                                      C.c_char_p, C.c_int]
            lib.tcref_session.restype = C.c_int
            lib.tcref_session.argtypes = [C.c_char_p, C.c_char_p, C.c_int, cpp, C.POINTER(C.c_int),
                                          C.POINTER(I64), C.c_uint64, C.c_int, cpp,
                                          C.POINTER(C.c_void_p), C.POINTER(I64), C.c_char_p, C.c_int]
            lib.tcref_options.restype = C.c_int
            lib.tcref_options.argtypes = [C.c_int, C.c_char_p, C.c_int, C.c_char_p, C.c_int]
            lib.tcref_options_roundtrip.restype = C.c_int
            lib.tcref_options_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_char_p,
                                                    C.c_int]
            lib.tcref_cache_serialize_one.restype = C.c_int
            lib.tcref_cache_serialize_one.argtypes = [C.c_char_p, C.c_char_p, C.c_int, cpp,
                                                      C.POINTER(C.c_int), C.POINTER(I64),
                                                      C.c_char_p, I64, I64, C.c_char_p, C.c_int,
                                                      C.c_char_p, C.c_int]
            lib.tcref_write_tensor.restype = C.c_int
            lib.tcref_write_tensor.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(I64), C.c_void_p,
                                               C.c_char_p, C.c_int]
            lib.tcref_read_tensor.restype = I64
            lib.tcref_read_tensor.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(I64),
                                              C.c_void_p, I64, C.c_char_p, C.c_int]
            RefLib._lib = lib
        self.lib = RefLib._lib

    @staticmethod
    def _names(names):
        arr = (C.c_char_p * len(names))(*[n.encode() for n in names])
        return C.cast(arr, C.POINTER(C.c_char_p)), arr

    @staticmethod
    def _shapes(shapes):
        ranks = (C.c_int * len(shapes))(*[len(s) for s in shapes])
        flat = [int(d) for s in shapes for d in s] or [0]
        return ranks, (I64 * len(flat))(*flat)

    def write_tensor(self, path, arr):
        """The reference's writeTensorFile (tensor_data.cc:122-147)."""
        a = np.ascontiguousarray(arr)
        shape = (I64 * max(1, a.ndim))(*a.shape)
        err = C.create_string_buffer(512)
        rc = self.lib.tcref_write_tensor(str(path).encode(), 1 if a.dtype == np.int32 else 0, a.ndim, shape,
                                         a.ctypes.data, err, 512)
        if rc:
            raise RefError(rc, err.value.decode())

    def read_tensor(self, path):
        """The reference's readTensorFile; raises RefError (kind Io) on malformed files."""
        kind, rank = C.c_int(), C.c_int()
        shape = (I64 * 16)()
        cap = 1 << 22
        buf = np.empty(cap, np.uint32)
        err = C.create_string_buffer(512)
        n = self.lib.tcref_read_tensor(str(path).encode(), C.byref(kind), C.byref(rank), shape,
                                       buf.ctypes.data, cap, err, 512)
        if n < 0:
            raise RefError(int(-n), err.value.decode())
        dt = np.int32 if kind.value else np.float32
        return buf[:n].view(dt).reshape(tuple(shape[d] for d in range(rank.value))).copy()

    def run(self, src, entry, inputs, out_names):
        """inputs: dict name -> np.ndarray (float32 or int32). Returns dict of outputs."""
        names = list(inputs)
        arrs = [np.ascontiguousarray(inputs[n]) for n in names]
        kinds = (C.c_int * len(names))(*[1 if a.dtype == np.int32 else 0 for a in arrs])
        ranks, flat = self._shapes([a.shape for a in arrs])
        datas = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        cap = 1 << 26
        outs = [np.empty(cap, np.float32) for _ in out_names]
        out_ptrs = (C.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
        caps = (I64 * len(outs))(*[cap] * len(outs))
        oshapes = (I64 * (8 * len(outs)))()
        oranks = (C.c_int * len(outs))()
        err = C.create_string_buffer(4096)
        nptr, _keep = self._names(names)
        onptr, _keep2 = self._names(out_names)
        rc = self.lib.tcref_run(src.encode(), entry.encode(), len(names), nptr, kinds, ranks, flat,
                                datas, len(out_names), onptr, out_ptrs, caps, oshapes, oranks,
                                err, 4096)
        if rc != 0:
            raise RefError(rc, err.value.decode())
        res = {}
        for i, n in enumerate(out_names):
            shape = tuple(oshapes[8 * i + d] for d in range(oranks[i]))
            res[n] = outs[i][: int(np.prod(shape))].reshape(shape).copy()
        return res

    def key(self, src, entry, shapes):
        names = list(shapes)
        ranks, flat = self._shapes([shapes[n] for n in names])
        canon = C.create_string_buffer(1 << 16)
        key = C.create_string_buffer(1 << 16)
        err = C.create_string_buffer(4096)
        nptr, _keep = self._names(names)
        rc = self.lib.tcref_key(src.encode(), entry.encode(), len(names), nptr, ranks, flat, canon,
                                1 << 16, key, 1 << 16, err, 4096)
        if rc != 0:
            raise RefError(rc, err.value.decode())
        return canon.value.decode(), key.value.decode()

    def session(self, src, entry, shapes, seed, out_names, kinds):
        names = list(shapes)
        ranks, flat = self._shapes([shapes[n] for n in names])
        outs = [np.empty(tuple(shapes[n]), np.int32 if kinds[n] else np.float32) for n in out_names]
        ptrs = (C.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
        caps = (I64 * len(outs))(*[o.size for o in outs])
        err = C.create_string_buffer(4096)
        nptr, _k = self._names(names)
        onptr, _k2 = self._names(out_names)
        rc = self.lib.tcref_session(src.encode(), entry.encode(), len(names), nptr, ranks, flat,
                                    seed, len(out_names), onptr, ptrs, caps, err, 4096)
        if rc != 0:
            raise RefError(rc, err.value.decode())
        return dict(zip(out_names, outs))

    def baseline_options(self):
        out = []
        i = 0
        while True:
            j = C.create_string_buffer(4096)
            d = C.create_string_buffer(64)
            if self.lib.tcref_options(i, j, 4096, d, 64) != 0:
                return out
            out.append((j.value.decode(), d.value.decode()))
            i += 1

    def options_roundtrip(self, text):
        o = C.create_string_buffer(4096)
        err = C.create_string_buffer(4096)
        rc = self.lib.tcref_options_roundtrip(text.encode(), o, 4096, err, 4096)
        if rc != 0:
            raise RefError(rc, err.value.decode())
        return o.value.decode()

    def cache_serialize_one(self, src, entry, shapes, options_json, cost, created_at):
        names = list(shapes)
        ranks, flat = self._shapes([shapes[n] for n in names])
        out = C.create_string_buffer(1 << 16)
        err = C.create_string_buffer(4096)
        nptr, _k = self._names(names)
        rc = self.lib.tcref_cache_serialize_one(src.encode(), entry.encode(), len(names), nptr,
                                                ranks, flat, options_json.encode(), cost,
                                                created_at, out, 1 << 16, err, 4096)
        if rc != 0:
            raise RefError(rc, err.value.decode())
        return out.value.decode()


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg
