"""Thin Python binding of libnfhmm's C-ABI (include/nfhmm.h): argument marshalling only.

Every step of the VB path runs in the library's sm_100a kernels.  There is no CPU fallback: if
libnfhmm.so is missing this module raises at import, and every call that fails on the device raises
NFHMMError with the library's status and message.

PyTorch is used for plumbing only: device memory (the workspace and any output tensors), the CUDA
stream handed to the library, and torch.distributed for multi-GPU sharding (bench.py).

The module-level functions carry the C names (nfhmm_create, nfhmm_set_model, ...); the NFHMM class
wraps a handle for convenience.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NFHMM_LIB") or os.path.join(_HERE, "lib", "libnfhmm.so")   # (override: A/B experiments)

NFHMM_OK, NFHMM_EINVAL, NFHMM_ESTATE, NFHMM_ECUDA = 0, -1, -2, -3
NFHMM_ENOMEM, NFHMM_EZEROSUPPORT, NFHMM_ENUMERIC = -4, -5, -6
MATH_TC, MATH_SIMT = 0, 1          # NFHMM_MATH_TC (tcgen05 3xTF32), NFHMM_MATH_SIMT (FP32 FFMA)


class NFHMMError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"libnfhmm status {status}: {msg}")
        self.status = status


class Options(ctypes.Structure):
    _fields_ = [("n_mix", ctypes.c_int64), ("gamma", ctypes.c_double), ("device", ctypes.c_int32),
                ("max_iters", ctypes.c_int32), ("free_energy", ctypes.c_int32), ("math", ctypes.c_int32),
                ("stream", ctypes.c_void_p)]


# symbol -> (restype, argtypes); mirrors include/nfhmm.h exactly (tests check the two agree)
_P, _I32, _I64, _D, _SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
SIGNATURES = {
    "nfhmm_default_options": (None, [ctypes.POINTER(Options)]),
    "nfhmm_create": (ctypes.c_int, [_I64, _I64, _I32, _I32, _I32, ctypes.POINTER(Options), ctypes.POINTER(_P)]),
    "nfhmm_workspace_size": (ctypes.c_int, [_P, ctypes.POINTER(_SZ)]),
    "nfhmm_set_workspace": (ctypes.c_int, [_P, _P, _SZ]),
    "nfhmm_set_model": (ctypes.c_int, [_P, _P, _P, _P]),
    "nfhmm_set_observations": (ctypes.c_int, [_P, _P]),
    "nfhmm_reset": (ctypes.c_int, [_P]),
    "nfhmm_vb_iterate": (ctypes.c_int, [_P, _I32]),
    "nfhmm_vb_iterate_async": (ctypes.c_int, [_P, _I32]),
    "nfhmm_sync": (ctypes.c_int, [_P]),
    "nfhmm_posteriors": (ctypes.c_int, [_P, _P, _P, _P, _P, ctypes.POINTER(_I32)]),
    "nfhmm_separate": (ctypes.c_int, [_P, _P, _P]),
    "nfhmm_separate_async": (ctypes.c_int, [_P, _P, _P]),
    "nfhmm_destroy": (ctypes.c_int, [_P]),
    "nfhmm_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "nfhmm_last_error": (ctypes.c_char_p, [_P]),
    "nfhmm_kernel_launches": (ctypes.c_int, [_P, ctypes.POINTER(_I64)]),
    "nfhmm_profile_enable": (ctypes.c_int, [_P, ctypes.c_int]),
    "nfhmm_profile_read": (ctypes.c_int, [_P, ctypes.POINTER(_D), ctypes.POINTER(_I64)]),
    "nfhmm_bench_kernel": (ctypes.c_int, [_P, ctypes.c_int, _I32, ctypes.POINTER(_D)]),
    "nfhmm_layout": (ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I32),
                                    ctypes.POINTER(_I32)]),
    "nfhmm_products": (ctypes.c_int, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "nfhmm_guard_check": (ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    # spectrogram front end / resynthesis
    "nfhmm_stft": (ctypes.c_int, [_P, _I64, _I64, _I32, _I32, ctypes.c_float, _P, _P, _I32, _P]),
    "nfhmm_istft": (ctypes.c_int, [_P, _P, _I64, _I32, _I64, _I32, _I32, ctypes.c_float, _P, _I64, _I32, _P]),
    # N-HMM EM training
    "nhmm_train_create": (ctypes.c_int, [_I64, _I64, _I32, _I32, _I64, _I32, _I32, _P, ctypes.POINTER(_P)]),
    "nhmm_train_set_data": (ctypes.c_int, [_P, _P]),
    "nhmm_train_set_params": (ctypes.c_int, [_P, _P, _P, _P, _P]),
    "nhmm_train_em": (ctypes.c_int, [_P, _I32]),
    "nhmm_train_get": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, ctypes.POINTER(_I32)]),
    "nhmm_train_kernel_launches": (ctypes.c_int, [_P, ctypes.POINTER(_I64)]),
    "nhmm_train_destroy": (ctypes.c_int, [_P]),
    "nhmm_train_last_error": (ctypes.c_char_p, [_P]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()


def library():
    return _lib


def _ptr(x):
    """Raw address of a numpy array / torch tensor (host or device); None -> NULL."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"], "arrays must be C-contiguous"
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous(), "tensors must be contiguous"
        return x.data_ptr()
    if isinstance(x, int):
        return x
    raise TypeError(f"unsupported array type {type(x)}")


def _check(h, status):
    if status != NFHMM_OK:
        msg = _lib.nfhmm_last_error(h).decode() if h else ""
        raise NFHMMError(status, msg or _lib.nfhmm_strerror(status).decode())


# ---- C-named thin wrappers ------------------------------------------------------------------
def nfhmm_default_options():
    o = Options()
    _lib.nfhmm_default_options(ctypes.byref(o))
    return o


def nfhmm_create(F, T, S, N, K, opt=None):
    h = ctypes.c_void_p()
    st = _lib.nfhmm_create(F, T, S, N, K, ctypes.byref(opt) if opt is not None else None, ctypes.byref(h))
    if st != NFHMM_OK:
        raise NFHMMError(st, _lib.nfhmm_strerror(st).decode())
    return h


def nfhmm_workspace_size(h):
    n = ctypes.c_size_t()
    _check(h, _lib.nfhmm_workspace_size(h, ctypes.byref(n)))
    return n.value


def nfhmm_set_workspace(h, dptr, nbytes):
    _check(h, _lib.nfhmm_set_workspace(h, dptr, nbytes))


def nfhmm_set_model(h, dict_, trans, prior):
    _check(h, _lib.nfhmm_set_model(h, _ptr(dict_), _ptr(trans), _ptr(prior)))


def nfhmm_set_observations(h, V):
    _check(h, _lib.nfhmm_set_observations(h, _ptr(V)))


def nfhmm_reset(h):
    _check(h, _lib.nfhmm_reset(h))


def nfhmm_vb_iterate(h, n_iters):
    _check(h, _lib.nfhmm_vb_iterate(h, n_iters))


def nfhmm_vb_iterate_async(h, n_iters):
    _check(h, _lib.nfhmm_vb_iterate_async(h, n_iters))


def nfhmm_sync(h):
    _check(h, _lib.nfhmm_sync(h))


def nfhmm_posteriors(h, d_hat=None, alpha_hat=None, V_hat=None, free_energy=None):
    it = ctypes.c_int32()
    _check(h, _lib.nfhmm_posteriors(h, _ptr(d_hat), _ptr(alpha_hat), _ptr(V_hat), _ptr(free_energy), ctypes.byref(it)))
    return it.value


def nfhmm_separate(h, V_star, V_src=None):
    _check(h, _lib.nfhmm_separate(h, _ptr(V_star), _ptr(V_src)))


def nfhmm_separate_async(h, V_star, V_src=None):
    _check(h, _lib.nfhmm_separate_async(h, _ptr(V_star), _ptr(V_src)))


def nfhmm_destroy(h):
    _lib.nfhmm_destroy(h)


def nfhmm_kernel_launches(h):
    n = ctypes.c_int64()
    _check(h, _lib.nfhmm_kernel_launches(h, ctypes.byref(n)))
    return n.value


def nfhmm_layout(h):
    fp, kp, br, bb = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
    _check(h, _lib.nfhmm_layout(h, ctypes.byref(fp), ctypes.byref(kp), ctypes.byref(br), ctypes.byref(bb)))
    return dict(F_pad=fp.value, Kt_pad=kp.value, bn_recon=br.value, bn_backproj=bb.value)


PRODUCTS = {0: "ffma", 1: "3xtf32", 2: "3xfp16"}


def nfhmm_products(h):
    """Product splitting of the (a) reconstruction and (b) back-projection contractions (include/nfhmm.h)."""
    r, b = ctypes.c_int32(), ctypes.c_int32()
    _check(h, _lib.nfhmm_products(h, ctypes.byref(r), ctypes.byref(b)))
    return dict(recon=PRODUCTS[r.value], backproj=PRODUCTS[b.value])


KERNEL_CLASSES = ("recon", "backproj", "dirichlet", "fb", "elbo", "separate", "other")


def nfhmm_guard_check(h):
    """(checked_bytes, bad_bytes) of the workspace guard zones (NFHMM_GUARD, include/nfhmm.h); returns
    rather than raises when zones were overwritten so the caller can report the counts."""
    c, b = ctypes.c_int64(), ctypes.c_int64()
    st = _lib.nfhmm_guard_check(h, ctypes.byref(c), ctypes.byref(b))
    if st not in (0, NFHMM_ECUDA) or (st == NFHMM_ECUDA and b.value == 0):
        _check(h, st)
    return c.value, b.value, (_lib.nfhmm_last_error(h).decode() if st else "")


def nfhmm_profile_enable(h, on=True):
    _check(h, _lib.nfhmm_profile_enable(h, 1 if on else 0))


def nfhmm_bench_kernel(h, cls, reps):
    """Mean device ms per launch of one kernel class run `reps` times back to back (ends with a reset)."""
    ms = ctypes.c_double()
    _check(h, _lib.nfhmm_bench_kernel(h, KERNEL_CLASSES.index(cls) if isinstance(cls, str) else cls, reps,
                                      ctypes.byref(ms)))
    return ms.value


def nfhmm_profile_read(h):
    """{class: (device ms, launches)} accumulated since the last enable (synchronises)."""
    n = len(KERNEL_CLASSES)
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_int64 * n)()
    _check(h, _lib.nfhmm_profile_read(h, ms, cnt))
    return {k: (ms[i], cnt[i]) for i, k in enumerate(KERNEL_CLASSES)}


# ---- convenience handle -----------------------------------------------------------------------
class NFHMM:
    """One libnfhmm handle: n_mix mixtures of F x T counts, S sources x N states x K elements.

    Inputs/outputs may be numpy arrays (host) or torch tensors (host or CUDA).  The workspace is a
    torch uint8 CUDA tensor owned by this object."""

    def __init__(self, F, T, S, N, K, n_mix=1, gamma=1.0, device=0, max_iters=1024, free_energy=True,
                 stream=None, math="tc"):
        import torch
        self.F, self.T, self.S, self.N, self.K, self.n_mix = F, T, S, N, K, n_mix
        self.Kt = S * N * K
        self.max_iters = max_iters
        self.device = device
        opt = nfhmm_default_options()
        opt.n_mix, opt.gamma, opt.device = n_mix, gamma, device
        opt.max_iters, opt.free_energy = max_iters, 1 if free_energy else 0
        opt.math = {"tc": MATH_TC, "simt": MATH_SIMT}[math]
        self.math = math
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        opt.stream = stream.cuda_stream
        self.h = nfhmm_create(F, T, S, N, K, opt)
        nbytes = nfhmm_workspace_size(self.h)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
        nfhmm_set_workspace(self.h, self.workspace.data_ptr(), nbytes)

    def close(self):
        if getattr(self, "h", None):
            nfhmm_destroy(self.h)
            self.h = None
        self.workspace = None   # the device memory goes back to torch's allocator with the handle

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_model(self, dict_, trans, prior):
        nfhmm_set_model(self.h, dict_, trans, prior)

    def set_observations(self, V):
        nfhmm_set_observations(self.h, V)

    def reset(self):
        nfhmm_reset(self.h)

    def vb_iterate(self, n):
        nfhmm_vb_iterate(self.h, n)

    def vb_iterate_async(self, n):
        nfhmm_vb_iterate_async(self.h, n)

    def sync(self):
        nfhmm_sync(self.h)

    def kernel_launches(self):
        return nfhmm_kernel_launches(self.h)

    def layout(self):
        return nfhmm_layout(self.h)

    def products(self):
        return nfhmm_products(self.h)

    def guard_check(self):
        return nfhmm_guard_check(self.h)

    def profile_enable(self, on=True):
        nfhmm_profile_enable(self.h, on)

    def profile_read(self):
        return nfhmm_profile_read(self.h)

    def bench_kernel(self, cls, reps=10):
        return nfhmm_bench_kernel(self.h, cls, reps)

    def posteriors(self, d_hat=True, alpha_hat=True, V_hat=True, free_energy=True):
        """Returns host numpy arrays: d_hat [M][S][T][N], alpha_hat [M][T][Kt], V_hat [M][T][F],
        free_energy [M][iters_done] (FP64), iters_done."""
        M, S, T, N, F, Kt = self.n_mix, self.S, self.T, self.N, self.F, self.Kt
        d = np.empty((M, S, T, N), np.float32) if d_hat else None
        a = np.empty((M, T, Kt), np.float32) if alpha_hat else None
        v = np.empty((M, T, F), np.float32) if V_hat else None
        fe = np.empty((M, self.max_iters), np.float64) if free_energy else None
        it = nfhmm_posteriors(self.h, d, a, v, fe)
        out = dict(iters_done=it)
        if d is not None:
            out["d_hat"] = d
        if a is not None:
            out["alpha_hat"] = a
        if v is not None:
            out["V_hat"] = v
        if fe is not None:
            out["free_energy"] = fe[:, :min(it, self.max_iters)]
        return out

    def separate_into(self, V_star, V_src=None, sync=True):
        """Separation into caller buffers (torch CUDA tensors, pinned host tensors or numpy arrays).
        sync=False: enqueue only (nfhmm_separate_async); read the outputs after sync()."""
        (nfhmm_separate if sync else nfhmm_separate_async)(self.h, V_star, V_src)

    def separate(self, V_src=False):
        M, S, T, F = self.n_mix, self.S, self.T, self.F
        vst = np.empty((M, S, T, F), np.float32)
        vs = np.empty((M, S, T, F), np.float32) if V_src else None
        nfhmm_separate(self.h, vst, vs)
        return (vst, vs) if V_src else vst


# ---- spectrogram front end / resynthesis (include/nfhmm.h nfhmm_stft / nfhmm_istft) ------

def _stream_ptr(stream, device):
    import torch
    if stream is None:
        return torch.cuda.current_stream(device).cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else stream


def stft(x, win=1024, hop=256, gain=1.0, device=0, stream=None, want_X=True, want_V=True):
    """x [n_sig][n_samples] float32 (numpy or torch) -> dict(X [n_sig][T][F] complex64, V [n_sig][T][F]),
    computed by libnfhmm's kernels (nfhmm_stft); outputs are host numpy arrays."""
    x = np.ascontiguousarray(x, np.float32) if isinstance(x, np.ndarray) else x
    if x.ndim == 1:
        x = x[None]
    n_sig, n = x.shape
    T, F = 1 + (n - win) // hop, win // 2 + 1
    X = np.empty((n_sig, T, F), np.complex64) if want_X else None
    V = np.empty((n_sig, T, F), np.float32) if want_V else None
    st = _lib.nfhmm_stft(_ptr(x), n_sig, n, win, hop, gain, _ptr(X), _ptr(V), device, _stream_ptr(stream, device))
    if st != NFHMM_OK:
        raise NFHMMError(st, _lib.nfhmm_strerror(st).decode())
    return dict(X=X, V=V)


def istft(X, M, n_samples, win=1024, hop=256, gain=1.0, device=0, stream=None):
    """X [n_mix][T][F] complex64 mixture STFT, M [n_mix][S][T][F] magnitudes in quanta -> y [n_mix][S][n_samples]
    (nfhmm_istft: the mixture's phase, weighted overlap-add)."""
    X = np.ascontiguousarray(X, np.complex64)
    M = np.ascontiguousarray(M, np.float32)
    n_mix, T, F = X.shape
    S = M.shape[1]
    y = np.empty((n_mix, S, n_samples), np.float32)
    st = _lib.nfhmm_istft(_ptr(X), _ptr(M), n_mix, S, T, win, hop, gain, _ptr(y), n_samples, device,
                          _stream_ptr(stream, device))
    if st != NFHMM_OK:
        raise NFHMMError(st, _lib.nfhmm_strerror(st).decode())
    return y


# ---- N-HMM EM training (include/nfhmm.h nhmm_train_*) --------------------------------

def _tcheck(h, status):
    if status != NFHMM_OK:
        msg = _lib.nhmm_train_last_error(h).decode() if h else ""
        raise NFHMMError(status, msg or _lib.nfhmm_strerror(status).decode())


class NHMMTrainer:
    """Maximum-likelihood EM for n_src independent single-source N-HMMs (argument marshalling only; the
    iteration runs in libnfhmm's kernels)."""

    def __init__(self, F, T, N, K, n_src=1, max_iters=256, device=0, stream=None):
        import torch
        self.F, self.T, self.N, self.K, self.n_src, self.max_iters = F, T, N, K, n_src, max_iters
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        h = ctypes.c_void_p()
        st = _lib.nhmm_train_create(F, T, N, K, n_src, max_iters, device, stream, ctypes.byref(h))
        if st != NFHMM_OK:
            raise NFHMMError(st, _lib.nfhmm_strerror(st).decode())
        self.h = h

    def set_data(self, V):
        _tcheck(self.h, _lib.nhmm_train_set_data(self.h, _ptr(V)))

    def set_params(self, dict_, trans, prior, weights=None):
        _tcheck(self.h, _lib.nhmm_train_set_params(self.h, _ptr(dict_), _ptr(trans), _ptr(prior), _ptr(weights)))

    def em(self, n_iters):
        _tcheck(self.h, _lib.nhmm_train_em(self.h, n_iters))

    def get(self):
        """Host numpy arrays: dict [n_src][N][K][F], trans [n_src][N][N], prior [n_src][N],
        weights [n_src][T][N][K], loglik [n_src][iters_done] (FP64)."""
        S, T, N, K, F = self.n_src, self.T, self.N, self.K, self.F
        d = np.empty((S, N, K, F), np.float32)
        tr = np.empty((S, N, N), np.float32)
        pr = np.empty((S, N), np.float32)
        w = np.empty((S, T, N, K), np.float32)
        ll = np.empty((S, self.max_iters), np.float64)
        it = ctypes.c_int32()
        _tcheck(self.h, _lib.nhmm_train_get(self.h, _ptr(d), _ptr(tr), _ptr(pr), _ptr(w), _ptr(ll), ctypes.byref(it)))
        return dict(dict=d, trans=tr, prior=pr, weights=w, loglik=ll[:, :it.value])

    def kernel_launches(self):
        n = ctypes.c_int64()
        _tcheck(self.h, _lib.nhmm_train_kernel_launches(self.h, ctypes.byref(n)))
        return n.value

    def close(self):
        if getattr(self, "h", None):
            _lib.nhmm_train_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
