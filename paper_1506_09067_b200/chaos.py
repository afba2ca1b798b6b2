"""Thin ctypes binding of libchaos.so (include/chaos.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels.  There is no CPU
fallback: if ``libchaos.so`` is missing or no CUDA device is present, construction
raises.  Names follow the C ABI (``chaos_net_create`` -> ``Net``, ``chaos_train_epoch``
-> ``Net.train_epoch`` ...).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# CHAOS_LIB selects the instrumented build (libchaos_timing.so) for profiling scripts
LIB_PATH = os.environ.get("CHAOS_LIB") or os.path.join(HERE, "libchaos.so")

CHAOS_CONV, CHAOS_MAXPOOL, CHAOS_FULL = 1, 2, 3
CHAOS_TANH, CHAOS_IDENTITY = 0, 1
HOGWILD, SYNC = 0, 1
OPT_STREAM, OPT_SYNC_BATCH, OPT_GROUP, OPT_MAX_CTAS, OPT_DEBUG_CLAIMS, OPT_RESERVE_SMS = 0, 1, 2, 3, 4, 5
OPT_DEBUG_TRACE, OPT_DEBUG_STAGGER, OPT_PAVG_COMM_CTAS = 6, 7, 8
TRACE_REC = 32  # int64 per group in chaos_debug_trace records
STATUS = {0: "CHAOS_OK", -1: "CHAOS_E_INVALID", -2: "CHAOS_E_ARCH", -3: "CHAOS_E_UNSUPPORTED",
          -4: "CHAOS_E_LABEL", -5: "CHAOS_E_NONFINITE", -6: "CHAOS_E_CUDA", -7: "CHAOS_E_NCCL"}

# every symbol include/chaos.h declares (checked by tests/test_abi.py)
EXPORTS = ["chaos_net_create", "chaos_net_destroy", "chaos_net_set_option", "chaos_net_get_option",
           "chaos_net_num_params", "chaos_net_get_params", "chaos_net_set_params", "chaos_net_device_params",
           "chaos_net_device_params_len", "chaos_train_epoch", "chaos_train_epoch_host", "chaos_last_train_loss",
           "chaos_evaluate", "chaos_forward", "chaos_compute_gradients", "chaos_debug_claims", "chaos_net_sync",
           "chaos_net_launch_info", "chaos_last_error", "chaos_last_status", "chaos_debug_phase_times",
           "chaos_batch_gradient", "chaos_apply_gradient", "chaos_progress_enqueued", "chaos_progress_wait",
           "chaos_avg_snapshot", "chaos_avg_apply", "chaos_dist_unique_id", "chaos_dist_init",
           "chaos_dist_average", "chaos_dist_average_buffer", "chaos_train_epoch_host_async", "chaos_debug_trace",
           "chaos_pavg_setup", "chaos_pavg_exchange", "chaos_pavg_ipc_handle", "chaos_pavg_open_peer",
           "chaos_pavg_set_peer", "chaos_pavg_arm", "chaos_pavg_rounds_done", "chaos_pavg_set_check",
           "chaos_pavg_debug_sums", "chaos_train_epoch_replicas"]
IPC_HANDLE_BYTES = 64


class ChaosError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Layer(C.Structure):
    _fields_ = [("kind", C.c_int32), ("units", C.c_int32), ("kernel", C.c_int32), ("act", C.c_int32)]


class Arch(C.Structure):
    _fields_ = [("in_c", C.c_int32), ("in_h", C.c_int32), ("in_w", C.c_int32), ("n_classes", C.c_int32),
                ("n_layers", C.c_int32), ("layers", Layer * 16), ("init_seed", C.c_uint64)]


_lib = None


def lib():
    """Load libchaos.so (raises if it was not built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        vp, fp, ip = C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_int32)
        sig = {
            "chaos_net_create": ([C.POINTER(Arch)], vp),
            "chaos_net_destroy": ([vp], None),
            "chaos_net_set_option": ([vp, C.c_int, C.c_int64], C.c_int),
            "chaos_net_get_option": ([vp, C.c_int], C.c_int64),
            "chaos_net_num_params": ([vp], C.c_int64),
            "chaos_net_get_params": ([vp, fp, C.c_int64], C.c_int),
            "chaos_net_set_params": ([vp, fp, C.c_int64], C.c_int),
            "chaos_net_device_params": ([vp], C.c_void_p),
            "chaos_net_device_params_len": ([vp], C.c_int64),
            "chaos_train_epoch": ([vp, vp, vp, C.c_int64, C.c_float, C.c_int], C.c_int),
            "chaos_train_epoch_host": ([vp, fp, ip, C.c_int64, C.c_float, C.c_int], C.c_int),
            "chaos_train_epoch_host_async": ([vp, fp, ip, C.c_int64, C.c_float, C.c_int], C.c_int),
            "chaos_last_train_loss": ([vp, C.POINTER(C.c_double)], C.c_int),
            "chaos_evaluate": ([vp, vp, vp, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int64)], C.c_int),
            "chaos_forward": ([vp, vp, C.c_int64, vp], C.c_int),
            "chaos_compute_gradients": ([vp, vp, vp, C.c_int64, fp], C.c_int),
            "chaos_debug_claims": ([vp, ip, C.c_int64], C.c_int),
            "chaos_debug_trace": ([vp, C.POINTER(C.c_int64), C.c_int64, fp, fp], C.c_int),
            "chaos_batch_gradient": ([vp, vp, vp, C.c_int64, vp], C.c_int),
            "chaos_apply_gradient": ([vp, vp, C.c_float], C.c_int),
            "chaos_net_sync": ([vp], C.c_int),
            "chaos_net_launch_info": ([vp, ip, ip, ip, ip], C.c_int),
            "chaos_last_error": ([], C.c_char_p),
            "chaos_last_status": ([], C.c_int),
            "chaos_debug_phase_times": ([vp, C.POINTER(C.c_uint64), C.c_int32], C.c_int),
            "chaos_progress_enqueued": ([vp], C.c_uint64),
            "chaos_progress_wait": ([vp, C.c_uint64, C.c_int64], C.c_int),
            "chaos_avg_snapshot": ([vp, vp, C.c_int64], C.c_int),
            "chaos_avg_apply": ([vp, vp, vp, C.c_int64], C.c_int),
            "chaos_dist_unique_id": ([vp], C.c_int),
            "chaos_dist_init": ([vp, vp, C.c_int32, C.c_int32], C.c_int),
            "chaos_dist_average": ([vp], C.c_int),
            "chaos_dist_average_buffer": ([vp, vp, C.c_int64, C.c_int64], C.c_int),
            "chaos_pavg_setup": ([vp, C.c_int32, C.c_int32, C.c_int64, C.c_int32], C.c_int),
            "chaos_pavg_exchange": ([vp, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)], C.c_int),
            "chaos_pavg_debug_sums": ([vp, fp, fp, C.c_int64], C.c_int),
            "chaos_pavg_ipc_handle": ([vp, vp], C.c_int),
            "chaos_pavg_open_peer": ([vp, C.c_int32, vp], C.c_int),
            "chaos_pavg_set_peer": ([vp, C.c_int32, vp], C.c_int),
            "chaos_pavg_arm": ([vp, C.c_int64], C.c_int),
            "chaos_pavg_rounds_done": ([vp], C.c_int64),
            "chaos_pavg_set_check": ([vp, C.c_int32], C.c_int),
            "chaos_train_epoch_replicas": ([C.POINTER(C.c_void_p), C.c_int32, C.POINTER(C.c_void_p),
                                            C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.c_float], C.c_int),
        }
        for name, (args, res) in sig.items():
            if os.environ.get("CHAOS_LIB") and not hasattr(L, name):
                continue  # an older library picked for an A/B experiment
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise ChaosError(rc, lib().chaos_last_error().decode())


def make_arch(layers, init_seed=0, in_c=1, in_h=29, in_w=29, n_classes=10) -> Arch:
    a = Arch()
    a.in_c, a.in_h, a.in_w, a.n_classes, a.n_layers = in_c, in_h, in_w, n_classes, len(layers)
    for i, (kind, units, kernel, act) in enumerate(layers):
        a.layers[i] = Layer(kind, units, kernel, act)
    a.init_seed = init_seed
    return a


def _ptr(t):
    """Device pointer of a CUDA torch tensor (contiguous)."""
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    return C.c_void_p(t.data_ptr())


def _check_batch(images, labels, n_in, device, cuda):
    """Images float32 with n * n_in elements, labels int32 of shape (n,), both on the net's device
    (cuda) or both host tensors/arrays (not cuda).  Raises ValueError (never stripped by -O)."""
    import torch
    n = int(labels.shape[0]) if labels is not None else int(images.shape[0])
    if isinstance(images, torch.Tensor):
        if images.dtype != torch.float32:
            raise ValueError(f"images must be float32, got {images.dtype}")
        if images.is_cuda != cuda or (cuda and images.device != device):
            raise ValueError(f"images must be on {device if cuda else 'the host'}, got {images.device}")
        if not images.is_contiguous():
            raise ValueError("images must be contiguous")
    numel = images.numel() if isinstance(images, torch.Tensor) else int(np.asarray(images).size)
    if numel != n * n_in:
        raise ValueError(f"images must hold n * {n_in} = {n * n_in} values for n = {n} labels")
    if labels is not None and isinstance(labels, torch.Tensor):
        if labels.dtype != torch.int32:
            raise ValueError(f"labels must be int32, got {labels.dtype}")
        if labels.is_cuda != cuda or (cuda and labels.device != device):
            raise ValueError(f"labels must be on {device if cuda else 'the host'}, got {labels.device}")
        if labels.dim() != 1 or not labels.is_contiguous():
            raise ValueError("labels must be a contiguous 1-D tensor")
    return n


class _CudaArray:
    """__cuda_array_interface__ wrapper so torch.as_tensor can alias the library's buffer."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "strides": None, "stream": None}


class Net:
    """chaos_net_create(arch) ... chaos_net_destroy."""

    def __init__(self, layers, init_seed=0, in_c=1, in_h=29, in_w=29, n_classes=10, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libchaos needs a CUDA device (no CPU fallback)")
        torch.cuda.init()
        self._arch = make_arch(layers, init_seed, in_c, in_h, in_w, n_classes)
        h = lib().chaos_net_create(C.byref(self._arch))
        if not h:
            raise ChaosError(lib().chaos_last_status(), lib().chaos_last_error().decode())
        self._h = C.c_void_p(h)
        self.n_params = int(lib().chaos_net_num_params(self._h))
        self.n_classes = n_classes
        self.n_in = in_c * in_h * in_w
        s = stream if stream is not None else torch.cuda.current_stream()
        self.set_option(OPT_STREAM, s.cuda_stream)
        self._stream = s
        self.device = torch.device("cuda", torch.cuda.current_device())

    def close(self):
        if getattr(self, "_h", None):
            lib().chaos_net_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self):
        return self._stream

    def set_option(self, opt, value):
        _check(lib().chaos_net_set_option(self._h, opt, int(value)))

    def get_option(self, opt):
        return int(lib().chaos_net_get_option(self._h, opt))

    def get_params(self) -> np.ndarray:
        out = np.zeros(self.n_params, np.float32)
        _check(lib().chaos_net_get_params(self._h, out.ctypes.data_as(C.POINTER(C.c_float)), self.n_params))
        return out

    def set_params(self, p):
        p = np.ascontiguousarray(p, np.float32)
        if p.shape != (self.n_params,):
            raise ValueError(f"expected {self.n_params} params")
        _check(lib().chaos_net_set_params(self._h, p.ctypes.data_as(C.POINTER(C.c_float)), self.n_params))

    def device_params(self):
        """torch view (no copy) of the internal parameter buffer (for NCCL averaging)."""
        import torch
        ptr = lib().chaos_net_device_params(self._h)
        n = int(lib().chaos_net_device_params_len(self._h))
        return torch.as_tensor(_CudaArray(ptr, n), device="cuda")

    def train_epoch(self, images, labels, lr, mode=HOGWILD):
        """chaos_train_epoch: asynchronous on the net's stream; images/labels CUDA tensors."""
        n = _check_batch(images, labels, self.n_in, self.device, True)
        _check(lib().chaos_train_epoch(self._h, _ptr(images), _ptr(labels), n, float(lr), int(mode)))

    def train_epoch_host(self, images, labels, lr, mode=HOGWILD):
        """chaos_train_epoch_host: host (ideally pinned) buffers; synchronizing."""
        import torch
        if isinstance(images, torch.Tensor):
            if not isinstance(labels, torch.Tensor):
                raise ValueError("images and labels must both be torch tensors or both numpy arrays")
            _check_batch(images, labels, self.n_in, None, False)
            xp = C.cast(C.c_void_p(images.data_ptr()), C.POINTER(C.c_float))
            yp = C.cast(C.c_void_p(labels.data_ptr()), C.POINTER(C.c_int32))
            n = int(labels.shape[0])
        else:
            images = np.ascontiguousarray(images, np.float32)
            labels = np.ascontiguousarray(labels, np.int32)
            if labels.ndim != 1 or images.size != len(labels) * self.n_in:
                raise ValueError(f"images must hold n * {self.n_in} values for n = {len(labels)} labels")
            xp = images.ctypes.data_as(C.POINTER(C.c_float))
            yp = labels.ctypes.data_as(C.POINTER(C.c_int32))
            n = len(labels)
        _check(lib().chaos_train_epoch_host(self._h, xp, yp, n, float(lr), int(mode)))

    def train_epoch_host_async(self, images, labels, lr, mode=HOGWILD):
        """chaos_train_epoch_host_async: pinned CPU torch tensors; returns once enqueued (the
        tensors are kept referenced until the next sync of this net)."""
        _check_batch(images, labels, self.n_in, None, False)
        # the library waits for a previous async epoch's copies before starting the next one, so
        # the tensors must stay referenced until then (and until sync())
        self._host_refs = getattr(self, "_host_refs", [])[-1:] + [(images, labels)]
        xp = C.cast(C.c_void_p(images.data_ptr()), C.POINTER(C.c_float))
        yp = C.cast(C.c_void_p(labels.data_ptr()), C.POINTER(C.c_int32))
        _check(lib().chaos_train_epoch_host_async(self._h, xp, yp, int(labels.shape[0]), float(lr), int(mode)))

    def last_train_loss(self):
        v = C.c_double()
        _check(lib().chaos_last_train_loss(self._h, C.byref(v)))
        return v.value

    def evaluate(self, images, labels):
        ml = C.c_double()
        ne = C.c_int64()
        n = _check_batch(images, labels, self.n_in, self.device, True)
        if n == 0:
            _check(lib().chaos_evaluate(self._h, None, None, 0, C.byref(ml), C.byref(ne)))
        else:
            _check(lib().chaos_evaluate(self._h, _ptr(images), _ptr(labels), n, C.byref(ml), C.byref(ne)))
        return ml.value, int(ne.value)

    def forward(self, images):
        import torch
        n = int(images.shape[0])
        _check_batch(images, None, self.n_in, self.device, True)
        out = torch.empty((n, self.n_classes), dtype=torch.float32, device=images.device)
        if n:
            _check(lib().chaos_forward(self._h, _ptr(images), n, _ptr(out)))
        return out

    def compute_gradients(self, images, labels):
        g = np.zeros(self.n_params, np.float32)
        n = _check_batch(images, labels, self.n_in, self.device, True)
        gp = g.ctypes.data_as(C.POINTER(C.c_float))
        if n == 0:
            _check(lib().chaos_compute_gradients(self._h, None, None, 0, gp))
        else:
            _check(lib().chaos_compute_gradients(self._h, _ptr(images), _ptr(labels), n, gp))
        return g

    def batch_gradient(self, images, labels, grad):
        """chaos_batch_gradient: grad (CUDA float32, device_params().numel()) = sum of the images'
        gradients at the current weights, internal layout; asynchronous on the net's stream."""
        n = _check_batch(images, labels, self.n_in, self.device, True)
        if grad.numel() != int(lib().chaos_net_device_params_len(self._h)) or grad.dtype.itemsize != 4:
            raise ValueError("grad must hold chaos_net_device_params_len float32 values")
        if n == 0:
            _check(lib().chaos_batch_gradient(self._h, None, None, 0, _ptr(grad)))
        else:
            _check(lib().chaos_batch_gradient(self._h, _ptr(images), _ptr(labels), n, _ptr(grad)))

    def apply_gradient(self, grad, lr):
        """chaos_apply_gradient: params -= lr * grad (internal layout); asynchronous."""
        _check(lib().chaos_apply_gradient(self._h, _ptr(grad), float(lr)))

    def progress_enqueued(self) -> int:
        """chaos_progress_enqueued: images enqueued to this net's hogwild launches so far."""
        return int(lib().chaos_progress_enqueued(self._h))

    def progress_wait(self, target, stream):
        """chaos_progress_wait on a torch.cuda.Stream other than the net's."""
        _check(lib().chaos_progress_wait(self._h, int(target), stream.cuda_stream))

    def avg_snapshot(self, snap, stream):
        _check(lib().chaos_avg_snapshot(self._h, _ptr(snap), stream.cuda_stream))

    def avg_apply(self, avg, snap, stream):
        """chaos_avg_apply: params += avg - snap (atomic, beside a running hogwild launch)."""
        _check(lib().chaos_avg_apply(self._h, _ptr(avg), _ptr(snap), stream.cuda_stream))

    @staticmethod
    def dist_unique_id() -> bytes:
        """chaos_dist_unique_id: 128 bytes to send from rank 0 to every rank."""
        buf = C.create_string_buffer(128)
        _check(lib().chaos_dist_unique_id(buf))
        return buf.raw

    def dist_init(self, uid: bytes, rank: int, world: int):
        """chaos_dist_init: the net's own NCCL communicator (collective)."""
        if len(uid) != 128:
            raise ValueError("expected the 128-byte id of dist_unique_id()")
        _check(lib().chaos_dist_init(self._h, C.create_string_buffer(uid, 128), int(rank), int(world)))

    def dist_average(self):
        """chaos_dist_average: params <- mean over the ranks, on the net's stream."""
        _check(lib().chaos_dist_average(self._h))

    def dist_average_buffer(self, buf, stream):
        """chaos_dist_average_buffer: in-place average of a CUDA float32 tensor on `stream`."""
        _check(lib().chaos_dist_average_buffer(self._h, _ptr(buf), int(buf.numel()), stream.cuda_stream))

    # ---- fused in-kernel cross-replica averaging (chaos_pavg_*; include/chaos.h)
    def pavg_setup(self, rank, world, k, nslice=0):
        """chaos_pavg_setup: this replica's exchange buffer (rank of world, interval k images)."""
        _check(lib().chaos_pavg_setup(self._h, int(rank), int(world), int(k), int(nslice)))
        self._pavg_rank = int(rank)

    def pavg_exchange(self, peer=None):
        """chaos_pavg_exchange: (device pointer, bytes) of rank `peer`'s exchange buffer as this net
        maps it (default: its own)."""
        p, b = C.c_void_p(), C.c_int64()
        if peer is None:
            peer = getattr(self, "_pavg_rank", None)
            if peer is None:
                raise ValueError("pavg_setup has not been called on this net")
        _check(lib().chaos_pavg_exchange(self._h, int(peer), C.byref(p), C.byref(b)))
        return int(p.value), int(b.value)

    def pavg_debug_sums(self):
        """chaos_pavg_debug_sums: (signed sum, magnitude sum) of the applied deltas (internal layout)."""
        n = int(lib().chaos_net_device_params_len(self._h))
        ds, da = np.zeros(n, np.float32), np.zeros(n, np.float32)
        fpp = C.POINTER(C.c_float)
        _check(lib().chaos_pavg_debug_sums(self._h, ds.ctypes.data_as(fpp), da.ctypes.data_as(fpp), n))
        return ds, da

    def pavg_ipc_handle(self) -> bytes:
        """chaos_pavg_ipc_handle: the exchange buffer's CUDA IPC handle (64 bytes)."""
        buf = C.create_string_buffer(IPC_HANDLE_BYTES)
        _check(lib().chaos_pavg_ipc_handle(self._h, buf))
        return buf.raw

    def pavg_open_peer(self, peer, handle: bytes):
        """chaos_pavg_open_peer: map rank `peer`'s exchange buffer (another process / GPU)."""
        if len(handle) != IPC_HANDLE_BYTES:
            raise ValueError(f"expected the {IPC_HANDLE_BYTES}-byte handle of pavg_ipc_handle()")
        _check(lib().chaos_pavg_open_peer(self._h, int(peer), C.create_string_buffer(handle, IPC_HANDLE_BYTES)))

    def pavg_set_peer(self, peer, other):
        """chaos_pavg_set_peer: another Net of this process (same device) is rank `peer`."""
        ptr, _ = other.pavg_exchange()
        _check(lib().chaos_pavg_set_peer(self._h, int(peer), C.c_void_p(ptr)))

    def pavg_arm(self, rounds):
        """chaos_pavg_arm: the next hogwild launch runs `rounds` in-kernel averaging rounds."""
        _check(lib().chaos_pavg_arm(self._h, int(rounds)))

    def pavg_rounds_done(self) -> int:
        return int(lib().chaos_pavg_rounds_done(self._h))

    def pavg_set_check(self, on=True):
        """chaos_pavg_set_check: debug checksums of every snapshot and every peer read of it."""
        _check(lib().chaos_pavg_set_check(self._h, 1 if on else 0))

    @staticmethod
    def train_epoch_replicas(nets, images, labels, lr):
        """chaos_train_epoch_replicas: one-GPU emulation, replica r = nets[r] trains images[r] /
        labels[r] (CUDA tensors) in ONE cooperative launch (asynchronous on nets[0]'s stream)."""
        R = len(nets)
        if not (len(images) == len(labels) == R):
            raise ValueError("one images / labels tensor per replica")
        ns = [_check_batch(x, y, nets[0].n_in, nets[0].device, True) for x, y in zip(images, labels)]
        hs = (C.c_void_p * R)(*[n._h.value for n in nets])
        xs = (C.c_void_p * R)(*[x.data_ptr() for x in images])
        ys = (C.c_void_p * R)(*[y.data_ptr() for y in labels])
        nn = (C.c_int64 * R)(*ns)
        _check(lib().chaos_train_epoch_replicas(hs, R, xs, ys, nn, float(lr)))

    def debug_trace(self, n_groups, pubs=True, reads=False):
        """chaos_debug_trace: (records int64 [n_groups][32], publishes float32 [n_groups][n_params]
        or None, weights read float32 [n_groups][2][n_params] or None; normative) of the last
        hogwild epoch run with OPT_DEBUG_TRACE = 1."""
        rec = np.zeros((n_groups, TRACE_REC), np.int64)
        pb = np.zeros((n_groups, self.n_params), np.float32) if pubs else None
        rd = np.zeros((n_groups, 2, self.n_params), np.float32) if reads else None
        fpp = C.POINTER(C.c_float)
        _check(lib().chaos_debug_trace(self._h, rec.ctypes.data_as(C.POINTER(C.c_int64)), n_groups,
                                       pb.ctypes.data_as(fpp) if pubs else None,
                                       rd.ctypes.data_as(fpp) if reads else None))
        return (rec, pb, rd) if reads else (rec, pb)

    def debug_claims(self, n):
        out = np.zeros(n, np.int32)
        _check(lib().chaos_debug_claims(self._h, out.ctypes.data_as(C.POINTER(C.c_int32)), n))
        return out

    PHASES = ["claim", "stage", "conv1_fwd", "conv2_fwd", "conv3_fwd", "fc_fwd", "loss", "fc2_bwd", "fc1_bwd",
              "conv3_din", "conv3_gw", "w2_load", "conv2_gw", "conv2_din", "img_reload", "conv1_gw",
              "fc1_fwd", "c3din_warps", "c3gw_warps", "p19"]

    def phase_times(self):
        """Per-phase clock64 cycles of the last hogwild epoch, summed over CTAs (timing build only)."""
        out = (C.c_uint64 * 20)()
        _check(lib().chaos_debug_phase_times(self._h, out, 20))
        return dict(zip(self.PHASES, [int(x) for x in out]))

    def sync(self):
        _check(lib().chaos_net_sync(self._h))
        self._host_refs = []

    def launch_info(self):
        v = [C.c_int32() for _ in range(4)]
        _check(lib().chaos_net_launch_info(self._h, *[C.byref(x) for x in v]))
        return {"grid": v[0].value, "block": v[1].value, "smem_bytes": v[2].value, "group": v[3].value}
