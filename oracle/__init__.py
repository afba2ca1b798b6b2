"""ctypes wrapper of the C oracle (``oracle/liboracle.so``).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path (``paper_1506_09067_b200``).
See ``oracle/oracle.h`` for the semantics and the PAPER.md passages each
function follows.  All parameters are float64, normative flat layout.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(HERE, "oracle.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", LIB_PATH, src, "-lm"])
    return LIB_PATH


class _Read(C.Structure):
    _fields_ = [("group", C.c_int32), ("layer", C.c_int32), ("purpose", C.c_int32), ("n_incl", C.c_int32),
                ("e0", C.c_int64), ("e1", C.c_int64), ("incl_off", C.c_int64)]


class _Layer(C.Structure):
    _fields_ = [("kind", C.c_int32), ("units", C.c_int32), ("kernel", C.c_int32), ("act", C.c_int32)]


class _Arch(C.Structure):
    _fields_ = [("in_c", C.c_int32), ("in_h", C.c_int32), ("in_w", C.c_int32), ("n_classes", C.c_int32),
                ("n_layers", C.c_int32), ("layers", _Layer * 16)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        fp = C.POINTER(C.c_float)
        ip = C.POINTER(C.c_int32)
        ap = C.POINTER(_Arch)
        _lib.orc_num_params.argtypes = [ap, C.c_char_p, C.c_int32]
        _lib.orc_num_params.restype = C.c_int64
        _lib.orc_blocks.argtypes = [ap, C.POINTER(C.c_int64), C.c_int32]
        _lib.orc_blocks.restype = C.c_int32
        _lib.orc_trace_len.argtypes = [ap]
        _lib.orc_trace_len.restype = C.c_int64
        _lib.orc_forward.argtypes = [ap, dp, fp, dp, dp, C.POINTER(C.c_uint8)]
        _lib.orc_sample_grad.argtypes = [ap, dp, fp, C.c_int32, dp, dp]
        _lib.orc_sample_grad2.argtypes = [ap, dp, dp, fp, C.c_int32, dp, dp]
        _lib.orc_replay.argtypes = [ap, dp, fp, ip, C.c_int32, C.POINTER(C.c_int64), ip, C.c_int32,
                                    C.POINTER(_Read), ip, C.c_double, dp, dp, dp]
        _lib.orc_train_sgd.argtypes = [ap, dp, fp, ip, C.c_int64, C.c_double, dp]
        _lib.orc_train_sync.argtypes = [ap, dp, fp, ip, C.c_int64, C.c_double, C.c_int64, dp]
        _lib.orc_evaluate.argtypes = [ap, dp, fp, ip, C.c_int64, dp, C.POINTER(C.c_int64), dp, ip]
        for f in ("orc_forward", "orc_sample_grad", "orc_sample_grad2", "orc_replay", "orc_train_sgd", "orc_train_sync", "orc_evaluate"):
            getattr(_lib, f).restype = C.c_int32
    return _lib


class OracleError(RuntimeError):
    pass


def make_arch(layers, in_c=1, in_h=29, in_w=29, n_classes=10) -> _Arch:
    a = _Arch()
    a.in_c, a.in_h, a.in_w, a.n_classes, a.n_layers = in_c, in_h, in_w, n_classes, len(layers)
    for i, (kind, units, kernel, act) in enumerate(layers):
        a.layers[i] = _Layer(kind, units, kernel, act)
    return a


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _check(rc):
    if rc != 0:
        raise OracleError(f"oracle returned {rc}")


class Oracle:
    """One architecture; every call is a pure function of its arguments."""

    def __init__(self, layers, in_c=1, in_h=29, in_w=29, n_classes=10):
        self.arch = make_arch(layers, in_c, in_h, in_w, n_classes)
        self.n_in = in_c * in_h * in_w
        self.n_classes = n_classes
        err = C.create_string_buffer(256)
        n = lib().orc_num_params(C.byref(self.arch), err, 256)
        if n < 0:
            raise OracleError(f"arch rejected ({n}): {err.value.decode()}")
        self.n_params = int(n)

    def blocks(self):
        out = (C.c_int64 * 48)()
        nl = lib().orc_blocks(C.byref(self.arch), out, 16)
        return [(int(out[3 * i]), int(out[3 * i + 1]), int(out[3 * i + 2])) for i in range(nl)]

    @staticmethod
    def _x(x):
        return np.ascontiguousarray(x, dtype=np.float32)

    @staticmethod
    def _p(p):
        return np.ascontiguousarray(p, dtype=np.float64)

    def forward(self, params, x):
        """Returns (logits[n_classes], trace[every layer output], argmax[u8 per pooled output])."""
        params = self._p(params)
        x = self._x(x)
        logits = np.zeros(self.n_classes)
        tl = lib().orc_trace_len(C.byref(self.arch))
        trace = np.zeros(tl)
        am = np.zeros(max(tl, 1), np.uint8)
        _check(lib().orc_forward(C.byref(self.arch), _d(params), _f(x), _d(logits), _d(trace),
                                 am.ctypes.data_as(C.POINTER(C.c_uint8))))
        return logits, trace, am

    def sample_grad(self, params, x, label):
        """Returns (loss, grad) of one sample."""
        params = self._p(params)
        x = self._x(x)
        g = np.zeros(self.n_params)
        loss = C.c_double()
        _check(lib().orc_sample_grad(C.byref(self.arch), _d(params), _f(x), int(label), _d(g), C.byref(loss)))
        return loss.value, g

    def sample_grad2(self, p_fwd, p_bwd, x, label):
        """(loss, grad) of one sample: forward at p_fwd, delta_in back-propagated at p_bwd."""
        pf, pb = self._p(p_fwd), self._p(p_bwd)
        x = self._x(x)
        g = np.zeros(self.n_params)
        loss = C.c_double()
        _check(lib().orc_sample_grad2(C.byref(self.arch), _d(pf), _d(pb), _f(x), int(label), _d(g), C.byref(loss)))
        return loss.value, g

    def replay(self, params0, X, Y, groups, reads, lr, pubs_in=None):
        """Hogwild schedule replay (orc_replay).  groups: [(first, count)]; reads: iterable of
        (group, layer, purpose, e0, e1, [included group ids]).  Returns (params, pubs[n_groups][P])."""
        p0 = self._p(params0)
        X = self._x(X)
        Y = np.ascontiguousarray(Y, np.int32)
        ng = len(groups)
        gf = np.ascontiguousarray([g[0] for g in groups], np.int64)
        gc = np.ascontiguousarray([g[1] for g in groups], np.int32)
        reads = list(reads)
        rd = (_Read * max(len(reads), 1))()
        incl = []
        for k, (grp, layer, purpose, e0, e1, inc) in enumerate(reads):
            rd[k] = _Read(grp, layer, purpose, len(inc), e0, e1, len(incl))
            incl.extend(int(j) for j in inc)
        inc = np.ascontiguousarray(incl if incl else [0], np.int32)
        out = np.zeros(self.n_params)
        pubs = np.zeros((max(ng, 1), self.n_params))
        pin = None if pubs_in is None else np.ascontiguousarray(pubs_in, np.float64)
        _check(lib().orc_replay(C.byref(self.arch), _d(p0), _f(X), _i(Y), ng,
                                gf.ctypes.data_as(C.POINTER(C.c_int64)), _i(gc), len(reads), rd, _i(inc),
                                float(lr), _d(out), _d(pubs), None if pin is None else _d(pin)))
        return out, pubs[:ng]

    def train_sgd(self, params, X, Y, lr):
        p = self._p(params).copy()
        X = self._x(X)
        Y = np.ascontiguousarray(Y, np.int32)
        s = C.c_double()
        _check(lib().orc_train_sgd(C.byref(self.arch), _d(p), _f(X), _i(Y), len(Y), lr, C.byref(s)))
        return p, s.value

    def train_sync(self, params, X, Y, lr, batch):
        p = self._p(params).copy()
        X = self._x(X)
        Y = np.ascontiguousarray(Y, np.int32)
        s = C.c_double()
        _check(lib().orc_train_sync(C.byref(self.arch), _d(p), _f(X), _i(Y), len(Y), lr, int(batch), C.byref(s)))
        return p, s.value

    def evaluate(self, params, X, Y, per_sample=False):
        params = self._p(params)
        X = self._x(X)
        Y = np.ascontiguousarray(Y, np.int32)
        n = len(Y)
        ml = C.c_double()
        ne = C.c_int64()
        losses = np.zeros(max(n, 1))
        preds = np.zeros(max(n, 1), np.int32)
        _check(lib().orc_evaluate(C.byref(self.arch), _d(params), _f(X), _i(Y), n, C.byref(ml), C.byref(ne),
                                  _d(losses), _i(preds)))
        if per_sample:
            return ml.value, int(ne.value), losses[:n], preds[:n]
        return ml.value, int(ne.value)
