"""paper_1004_3105_b200 -- B200-native bulk fp64 normal generators (Brent 1993: B1/B2/B3, Polar).

Thin Python binding over the C ABI of ``libnrng.so`` (``include/nrng.h``):
argument marshalling only.  Every step of the method runs in the sm_100a kernels;
PyTorch supplies device memory, CUDA streams and process groups.  There is no CPU
fallback: if ``libnrng.so`` is missing or no CUDA device is usable, calls raise.

The low-level functions carry the C names (``nrng_create``, ``nrng_normal_boxmuller``,
...).  ``Generator`` wraps a handle for torch users.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NRNG_LIB_OVERRIDE") or os.path.join(PKG, "libnrng.so")  # override: A/B builds only

NRNG_DEFAULT, NRNG_B1, NRNG_B2, NRNG_B3, NRNG_POLAR, NRNG_POLAR2 = 0, 1, 2, 3, 4, 5
NRNG_OK, NRNG_EINVAL, NRNG_ENOMEM, NRNG_ECUDA, NRNG_ENODEV = 0, -1, -2, -3, -4
LAG_R = 607
METHODS = {"B1": 1, "B2": 2, "B3": 3, "P": 4, "P2": 5, "R": 6, "R1": 7}

# name -> (argtypes, restype); mirrors include/nrng.h one to one
_u64, _u32, _dbl, _p, _int, _sz = C.c_uint64, C.c_uint32, C.c_double, C.c_void_p, C.c_int, C.c_size_t
SIGNATURES = {
    "nrng_create": ([_u64, _u32, _int], _p),
    "nrng_create_range": ([_u64, _u64, _u32, _int], _p),
    "nrng_destroy": ([_p], None),
    "nrng_set_stream": ([_p, _p], _int),
    "nrng_normal_boxmuller": ([_p, _p, _sz, _dbl, _dbl, _int], _int),
    "nrng_normal_polar": ([_p, _p, _sz, _dbl, _dbl], _int),
    "nrng_normal_polar2": ([_p, _p, _sz, _dbl, _dbl], _int),
    "nrng_normal_ratio": ([_p, _p, _sz, _dbl, _dbl], _int),
    "nrng_normal_ratio1": ([_p, _p, _sz, _dbl, _dbl], _int),
    "nrng_serial_corr": ([_p, _sz, _dbl, _int, _p, _p], _int),
    "nrng_serial_corr_blocks": ([_sz], _sz),
    "nrng_seq_configure": ([_p, _u32], _int),
    "nrng_normal_seq": ([_p, _p, _sz, _dbl, _dbl, _int], _int),
    "nrng_seq_buffered": ([_p], _sz),
    "nrng_seq_reset": ([_p], _int),
    "nrng_last_error": ([], _int),
    "nrng_error_string": ([_int], C.c_char_p),
    "nrng_num_streams": ([_p], _u32),
    "nrng_first_stream": ([_p], _u64),
    "nrng_stream_counts": ([_p, _p], _int),
    "nrng_get_state": ([_p, _p, _p], _int),
    "nrng_set_state": ([_p, _p, _p], _int),
    "nrng_synchronize": ([_p], _int),
    "nrng_kernel_launches": ([_p], _u64),
    "nrng_racecheck_result": ([_p], _int),
    "nrng_uniform": ([_p, _p, _sz], _int),
    "nrng_polar_mask": ([_p, _p, _sz], _int),
    "nrng_transform_from_uniforms": ([_p, _sz, _p, _p, _dbl, _dbl, _int, _p], _int),
    "nrng_stats": ([_p, _sz, _dbl, _p, _int, _p, _p, _p], _int),
    "nrng_gof_hist": ([_p, _sz, _dbl, _dbl, _int, _p, _p], _int),
}

_lib = None


class NrngError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__("%s failed: %s (%d)" % (what, _errstr(code), code))
        self.code = code


def lib():
    """Load libnrng.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libnrng.so not built: run `python -m paper_1004_3105_b200.build` "
                              "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            if os.environ.get("NRNG_LIB_OVERRIDE") and not hasattr(L, name):
                continue  # an older A/B build without a newer entry point
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _errstr(code: int) -> str:
    try:
        return lib().nrng_error_string(code).decode()
    except Exception:  # pragma: no cover
        return "error"


def _check(rc: int, what: str) -> None:
    if rc != NRNG_OK:
        raise NrngError(rc, what)


# ------------------------------------------------------------------ C-named wrappers
def nrng_create(seed: int, n_streams: int, variant: int = 0) -> int:
    h = lib().nrng_create(seed, n_streams, variant)
    if not h:
        raise NrngError(lib().nrng_last_error(), "nrng_create")
    return h


def nrng_create_range(seed: int, first_stream: int, n_streams: int, variant: int = 0) -> int:
    h = lib().nrng_create_range(seed, first_stream, n_streams, variant)
    if not h:
        raise NrngError(lib().nrng_last_error(), "nrng_create_range")
    return h


def nrng_destroy(h) -> None:
    lib().nrng_destroy(h)


def nrng_set_stream(h, cuda_stream: int) -> None:
    _check(lib().nrng_set_stream(h, cuda_stream), "nrng_set_stream")


def nrng_normal_boxmuller(h, out_ptr: int, n: int, mu: float, sigma: float, variant: int = 0) -> None:
    _check(lib().nrng_normal_boxmuller(h, out_ptr, n, mu, sigma, variant), "nrng_normal_boxmuller")


def nrng_normal_polar(h, out_ptr: int, n: int, mu: float, sigma: float) -> None:
    _check(lib().nrng_normal_polar(h, out_ptr, n, mu, sigma), "nrng_normal_polar")


def nrng_normal_polar2(h, out_ptr: int, n: int, mu: float, sigma: float) -> None:
    _check(lib().nrng_normal_polar2(h, out_ptr, n, mu, sigma), "nrng_normal_polar2")


def nrng_normal_ratio(h, out_ptr: int, n: int, mu: float, sigma: float) -> None:
    _check(lib().nrng_normal_ratio(h, out_ptr, n, mu, sigma), "nrng_normal_ratio")


def nrng_normal_ratio1(h, out_ptr: int, n: int, mu: float, sigma: float) -> None:
    _check(lib().nrng_normal_ratio1(h, out_ptr, n, mu, sigma), "nrng_normal_ratio1")


def nrng_seq_configure(h, epoch_pairs: int) -> None:
    _check(lib().nrng_seq_configure(h, epoch_pairs), "nrng_seq_configure")


def nrng_normal_seq(h, out_ptr: int, n: int, mu: float, sigma: float, method: int) -> None:
    _check(lib().nrng_normal_seq(h, out_ptr, n, mu, sigma, method), "nrng_normal_seq")


def nrng_seq_buffered(h) -> int:
    return int(lib().nrng_seq_buffered(h))


def nrng_seq_reset(h) -> None:
    _check(lib().nrng_seq_reset(h), "nrng_seq_reset")


def nrng_uniform(h, out_ptr: int, n: int) -> None:
    _check(lib().nrng_uniform(h, out_ptr, n), "nrng_uniform")


def nrng_polar_mask(h, mask_ptr: int, cand_per_stream: int) -> None:
    _check(lib().nrng_polar_mask(h, mask_ptr, cand_per_stream), "nrng_polar_mask")


def nrng_transform_from_uniforms(u_ptr, n_pairs, out_ptr, mask_ptr, mu, sigma, method, stream) -> None:
    _check(lib().nrng_transform_from_uniforms(u_ptr, n_pairs, out_ptr, mask_ptr, mu, sigma, method, stream),
           "nrng_transform_from_uniforms")


def nrng_stats(x_ptr, n, center, edges_ptr, K, sums_ptr, hist_ptr, stream) -> None:
    _check(lib().nrng_stats(x_ptr, n, center, edges_ptr, K, sums_ptr, hist_ptr, stream), "nrng_stats")


def nrng_gof_hist(x_ptr, n, mu, sigma, log2K, hist_ptr, stream) -> None:
    _check(lib().nrng_gof_hist(x_ptr, n, mu, sigma, log2K, hist_ptr, stream), "nrng_gof_hist")


def nrng_serial_corr(x_ptr, n, center, K, partial_ptr, stream) -> None:
    _check(lib().nrng_serial_corr(x_ptr, n, center, K, partial_ptr, stream), "nrng_serial_corr")


def nrng_serial_corr_blocks(n: int) -> int:
    return int(lib().nrng_serial_corr_blocks(n))


def nrng_last_error() -> int:
    return lib().nrng_last_error()


def nrng_error_string(code: int) -> str:
    return _errstr(code)


def nrng_num_streams(h) -> int:
    return lib().nrng_num_streams(h)


def nrng_first_stream(h) -> int:
    return lib().nrng_first_stream(h)


def nrng_synchronize(h) -> None:
    _check(lib().nrng_synchronize(h), "nrng_synchronize")


def nrng_kernel_launches(h) -> int:
    return int(lib().nrng_kernel_launches(h))


def nrng_racecheck_result():
    """(races, first race code, accesses checked) of a NRNG_RACECHECK debug build; raises
    NrngError(EINVAL) on the product build."""
    out = np.zeros(3, np.uint64)
    _check(lib().nrng_racecheck_result(out.ctypes.data), "nrng_racecheck_result")
    return int(out[0]), int(out[1]), int(out[2])


def nrng_stream_counts(h) -> np.ndarray:
    out = np.empty(nrng_num_streams(h), np.uint64)
    _check(lib().nrng_stream_counts(h, out.ctypes.data), "nrng_stream_counts")
    return out


def nrng_get_state(h):
    S = nrng_num_streams(h)
    ring = np.empty((S, LAG_R), np.uint64)
    cnt = np.empty(S, np.uint64)
    _check(lib().nrng_get_state(h, ring.ctypes.data, cnt.ctypes.data), "nrng_get_state")
    return ring, cnt


def nrng_set_state(h, ring: np.ndarray, counts: np.ndarray) -> None:
    ring = np.ascontiguousarray(ring, np.uint64)
    counts = np.ascontiguousarray(counts, np.uint64)
    _check(lib().nrng_set_state(h, ring.ctypes.data, counts.ctypes.data), "nrng_set_state")


# ------------------------------------------------------------------ torch-facing API
def _torch():
    import torch

    return torch


def _stream_ptr(torch):
    # the raw cudaStream_t of torch's current stream; the private accessor skips building a
    # torch.cuda.Stream object (3 us of the ~10 us host cost of a short call, measured)
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def out_buffer(out, device=None):
    """(pointer, number of doubles) of a caller's output buffer, after checking that the
    library may write 8 * size bytes there: float64, C-contiguous, and -- for a CUDA tensor --
    on the handle's device (`device`, a torch.device).  A numpy array or CPU tensor is a host
    buffer (the library's host-output path).  Raises TypeError / ValueError otherwise."""
    if isinstance(out, np.ndarray):
        if out.dtype != np.float64:
            raise TypeError("out must be float64, got %s" % out.dtype)
        if not out.flags.c_contiguous or not out.flags.writeable:
            raise ValueError("out must be a writeable C-contiguous array")
        return out.ctypes.data, out.size
    torch = _torch()
    if not isinstance(out, torch.Tensor):
        raise TypeError("out must be a torch tensor or a numpy array, got %s" % type(out).__name__)
    if out.dtype != torch.float64:
        raise TypeError("out must be float64, got %s" % out.dtype)
    if not out.is_contiguous():
        raise ValueError("out must be contiguous")
    if out.device.type == "cuda":
        if device is not None and out.device != torch.device(device):
            raise ValueError("out is on %s but the generator lives on %s" % (out.device, device))
    elif out.device.type != "cpu":
        raise ValueError("out must be a CUDA or CPU tensor, got %s" % out.device)
    return out.data_ptr(), out.numel()


class Generator:
    """A set of LFG streams [first_stream, first_stream + n_streams) on the current CUDA device.

    Outputs are torch float64 tensors (device by default) or caller buffers: a CUDA
    tensor, or a CPU tensor / numpy array (the library's host-output path).
    """

    def __init__(self, seed: int, n_streams: int, variant: int = 1, first_stream: int = 0):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1004_3105_b200 needs a CUDA device (no CPU fallback)")
        self.seed, self.S, self.first, self.variant = int(seed), int(n_streams), int(first_stream), int(variant)
        self._dev = torch.cuda.current_device()
        self.device = torch.device("cuda", self._dev)
        self.h = nrng_create_range(self.seed, self.first, self.S, self.variant)
        self._torch = torch
        raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
        self._raw_stream = (lambda: raw(self._dev)) if raw is not None else (
            lambda: torch.cuda.current_stream(self._dev).cuda_stream)
        self._stream = self._raw_stream()
        nrng_set_stream(self.h, self._stream)
        L = lib()
        # per method: (C entry point, trailing arguments, name for errors); the short-call path
        # below costs a few microseconds of host time per call, so it avoids per-call lookups
        bm = L.nrng_normal_boxmuller
        self._calls = {"B1": (bm, (1,)), "B2": (bm, (2,)), "B3": (bm, (3,)),
                       "P": (L.nrng_normal_polar, ()), "P2": (L.nrng_normal_polar2, ()),
                       "R": (L.nrng_normal_ratio, ()), "R1": (L.nrng_normal_ratio1, ())}

    def close(self):
        if getattr(self, "h", None):
            nrng_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def _sync_stream(self):
        sp = self._raw_stream()
        if sp != self._stream:  # the handle keeps its stream: only tell it about changes
            nrng_set_stream(self.h, sp)
            self._stream = sp

    def _out(self, n, out):
        torch = self._torch
        if out is None:
            out = torch.empty(n, dtype=torch.float64, device=self.device)
            return out, out.data_ptr(), n
        if type(out) is torch.Tensor and out.is_cuda:  # fast path of out_buffer's checks
            if out.dtype is not torch.float64 or not out.is_contiguous() or out.get_device() != self._dev:
                out_buffer(out, self.device)  # raises with the reason
            return out, out.data_ptr(), out.numel()
        ptr, size = out_buffer(out, self.device)
        return out, ptr, size

    def _call(self, key, n, mu, sigma, out):
        fn, extra = self._calls[key]
        out, ptr, n = self._out(n, out)
        self._sync_stream()
        rc = fn(self.h, ptr, n, mu, sigma, *extra)
        if rc:
            raise NrngError(rc, fn.__name__)
        return out

    def normal_boxmuller(self, n: int = None, mu: float = 0.0, sigma: float = 1.0, variant: int = 0, out=None):
        out, ptr, n = self._out(n, out)
        self._sync_stream()
        nrng_normal_boxmuller(self.h, ptr, n, mu, sigma, variant)
        return out

    def normal_polar(self, n: int = None, mu: float = 0.0, sigma: float = 1.0, out=None):
        return self._call("P", n, mu, sigma, out)

    def normal_polar2(self, n: int = None, mu: float = 0.0, sigma: float = 1.0, out=None):
        return self._call("P2", n, mu, sigma, out)

    def normal_ratio(self, n: int = None, mu: float = 0.0, sigma: float = 1.0, out=None):
        """Algorithm R (the ratio method): one normal per accepted candidate."""
        return self._call("R", n, mu, sigma, out)

    def normal_ratio1(self, n: int = None, mu: float = 0.0, sigma: float = 1.0, out=None):
        """Algorithm R1 (R with the step-2.5 pretests): the same output as normal_ratio."""
        return self._call("R1", n, mu, sigma, out)

    def normal(self, method: str, n: int = None, mu: float = 0.0, sigma: float = 1.0, out=None):
        """n deviates of N(mu, sigma^2) by `method` (B1, B2, B3, P, P2, R, R1) into `out` (a new
        CUDA tensor by default; a CUDA tensor, CPU tensor or numpy array otherwise)."""
        return self._call(method, n, mu, sigma, out)

    def normal_seq(self, method: str, n: int = None, mu: float = 0.0, sigma: float = 1.0, out=None):
        """Next n deviates of the handle's canonical sequence (RANN3-style buffering)."""
        out, ptr, n = self._out(n, out)
        self._sync_stream()
        nrng_normal_seq(self.h, ptr, n, mu, sigma, METHODS[method])
        return out

    def uniform(self, n: int = None, out=None):
        out, ptr, n = self._out(n, out)
        self._sync_stream()
        nrng_uniform(self.h, ptr, n)
        return out

    def polar_mask(self, cand_per_stream: int):
        torch = _torch()
        m = torch.empty(self.S * cand_per_stream, dtype=torch.uint8, device=self.device)
        self._sync_stream()
        nrng_polar_mask(self.h, m.data_ptr(), cand_per_stream)
        return m

    def stream_counts(self) -> np.ndarray:
        return nrng_stream_counts(self.h)

    def get_state(self):
        return nrng_get_state(self.h)

    def set_state(self, ring, counts):
        nrng_set_state(self.h, ring, counts)

    def synchronize(self):
        nrng_synchronize(self.h)

    @property
    def kernel_launches(self) -> int:
        return nrng_kernel_launches(self.h)


def _device_f64(x, what="x"):
    """A contiguous float64 CUDA tensor for the device-side hooks (raises otherwise)."""
    torch = _torch()
    if not isinstance(x, torch.Tensor) or x.dtype != torch.float64 or x.device.type != "cuda":
        raise TypeError("%s must be a float64 CUDA tensor" % what)
    if not x.is_contiguous():
        raise ValueError("%s must be contiguous" % what)
    return x


def transform_from_uniforms(u, method: int, mu: float = 0.0, sigma: float = 1.0):
    """Device transform on given uniforms: method 1/2/3 = B1/B2/B3, 4 = Polar, 5 = P2, 6 = R, 7 = R1.
    Returns (out, mask)."""
    torch = _torch()
    _device_f64(u, "u")
    per = 3 if method == 3 else 2
    n_pairs = u.numel() // per
    out = torch.empty(2 * n_pairs, dtype=torch.float64, device=u.device)
    mask = torch.empty(n_pairs, dtype=torch.uint8, device=u.device) if method >= 4 else None
    nrng_transform_from_uniforms(u.data_ptr(), n_pairs, out.data_ptr(), mask.data_ptr() if mask is not None else None,
                                 mu, sigma, method, _stream_ptr(torch))
    return out, mask


def serial_corr(x, center: float, K: int = 100):
    """Device lagged sums S_k = sum_i (x_i - c)(x_{i+k} - c), k = 0..K, summed over blocks in a
    fixed order (numpy float64 array of K+1)."""
    torch = _torch()
    _device_f64(x)
    n = x.numel()
    nb = nrng_serial_corr_blocks(n)
    part = torch.empty(max(1, nb) * (K + 1), dtype=torch.float64, device=x.device)
    nrng_serial_corr(x.data_ptr(), n, center, K, part.data_ptr(), _stream_ptr(torch))
    if nb == 0:
        return np.zeros(K + 1)
    return part.view(nb, K + 1).cpu().numpy().sum(axis=0)


def stats(x, center: float, edges):
    """Device validation reduction: (sums[6] = sum d, d^2, d^3, d^4, min, max; hist[K] int64)."""
    torch = _torch()
    _device_f64(x)
    edges = torch.as_tensor(edges, dtype=torch.float64, device=x.device).contiguous()
    K = edges.numel() + 1
    sums = torch.empty(6, dtype=torch.float64, device=x.device)
    hist = torch.empty(K, dtype=torch.int64, device=x.device)
    nrng_stats(x.data_ptr(), x.numel(), center, edges.data_ptr(), K, sums.data_ptr(), hist.data_ptr(),
               _stream_ptr(torch))
    return sums, hist


def gof_hist(x, mu: float, sigma: float, log2K: int = 20):
    """Device histogram of Phi((x-mu)/sigma) over 2^log2K equal-probability bins (int32 tensor)."""
    torch = _torch()
    _device_f64(x)
    hist = torch.empty(1 << log2K, dtype=torch.int32, device=x.device)
    nrng_gof_hist(x.data_ptr(), x.numel(), mu, sigma, log2K, hist.data_ptr(), _stream_ptr(torch))
    return hist
