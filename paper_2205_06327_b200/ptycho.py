"""Thin Python binding of include/ptycho.h (ctypes; argument marshalling only).

Every step of the hot path runs in libptycho.so's sm_100a kernels.  There is no CPU or
PyTorch fallback: if the extension is missing, importing this module raises.  PyTorch is used
only for device memory (the workspace), streams and torch.distributed plumbing.

The raw C entry points are exported under their C names (ptycho_create, ptycho_set_tiles, ...);
the class `Ptycho` wraps them for tests and bench.py.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PTYCHO_LIB", os.path.join(_HERE, "lib", "libptycho.so"))  # override: A/B builds

PTYCHO_F_EXACT_WINDOW = 1
PTYCHO_F_STASH_FREE = 2
PTYCHO_APPP_AUTO, PTYCHO_APPP_NCCL, PTYCHO_APPP_P2P = 0, 1, 2
PTYCHO_AMP_DC_CENTERED = 1
PTYCHO_AMP_INTENSITY = 2
PTYCHO_AMP_ASYNC = 4
STATUS = {0: "OK", 1: "EARG", 2: "ESHAPE", 3: "ESTATE", 4: "EHALO", 5: "ECUDA", 6: "ENCCL", 7: "ENOMEM"}


class ptycho_config(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("slices", ctypes.c_int32), ("height", ctypes.c_int32),
                ("width", ctypes.c_int32), ("sigma", ctypes.c_float), ("prop_c", ctypes.c_float),
                ("alpha", ctypes.c_float), ("alpha_acc", ctypes.c_float), ("tau", ctypes.c_float),
                ("pass_period", ctypes.c_int32), ("flags", ctypes.c_int32)]


if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the CUDA extension is required; there is no fallback)")
lib = ctypes.CDLL(LIB_PATH)

_c = ctypes
_P = _c.c_void_p
_SIGS = {
    "ptycho_create": [_c.POINTER(ptycho_config), _c.c_int, _P, _c.POINTER(_P)],
    "ptycho_destroy": [_P],
    "ptycho_nccl_unique_id": [_P, _c.c_size_t],
    "ptycho_set_tiles": [_P, _c.c_int32, _c.c_int32, _c.c_int32, _P, _P, _c.c_int32, _c.c_int32],
    "ptycho_set_tiles_hve": [_P, _c.c_int32, _c.c_int32, _c.c_int32, _c.c_int32, _P, _P, _c.c_int32, _c.c_int32],
    "ptycho_set_scan": [_P, _P, _c.c_int64],
    "ptycho_tile_geometry": [_c.c_int32, _c.c_int32, _c.c_int32, _c.c_int32, _c.c_int32, _P],
    "ptycho_appp_schedule": [_c.c_int32, _c.c_int32, _c.c_int32, _c.c_int32, _c.c_int32, _P, _c.c_int32,
                             _c.POINTER(_c.c_int32)],
    "ptycho_local_probes": [_P, _P, _c.POINTER(_c.c_int64)],
    "ptycho_tile_probe_count": [_P, _c.c_int32, _c.POINTER(_c.c_int64)],
    "ptycho_tile_rect": [_P, _c.c_int32, _P, _P],
    "ptycho_set_schedule": [_P, _c.c_int32, _c.c_int32],
    "ptycho_workspace_bytes": [_P, _c.POINTER(_c.c_size_t)],
    "ptycho_set_workspace": [_P, _P, _c.c_size_t],
    "ptycho_set_probe": [_P, _P, _c.c_int],
    "ptycho_load_measurements": [_P, _P, _c.c_int, _c.c_int64, _c.c_int64, _c.c_int32],
    "ptycho_read_measurements": [_P, _P, _c.c_int64, _c.c_int64],
    "ptycho_set_volume": [_P, _P, _c.c_int],
    "ptycho_simulate_measurements": [_P],
    "ptycho_forward_grad": [_P, _c.c_int64, _c.c_int64, _c.POINTER(_c.c_double)],
    "ptycho_appp_passes": [_P],
    "ptycho_set_appp_transport": [_P, _c.c_int32],
    "ptycho_appp_transport": [_P, _c.POINTER(_c.c_int32)],
    "ptycho_step": [_P],
    "ptycho_iterate": [_P, _c.POINTER(_c.c_double)],
    "ptycho_stitch": [_P, _P, _c.c_int, _c.c_int32],
    "ptycho_synchronize": [_P],
    "ptycho_kernel_launches": [_P, _c.POINTER(_c.c_int64)],
    "ptycho_profile_chain": [_P, _c.c_int32, _c.c_int64, _c.c_int64, _P, _P],
    "ptycho_profile_iteration": [_P, _P],
    "ptycho_debug_errors": [_P, _P, _P],
    "ptycho_debug_read_tile": [_P, _c.c_int32, _c.c_int32, _P],
    "ptycho_debug_write_tile": [_P, _c.c_int32, _c.c_int32, _P],
    "ptycho_debug_probe_grad": [_P, _c.c_int32, _c.c_int64, _P, _c.POINTER(_c.c_double)],
    "ptycho_debug_exit_wave": [_P, _c.c_int32, _c.c_int64, _P],
    "ptycho_probe_grad": [_P, _c.c_int64, _P, _c.POINTER(_c.c_double)],
    "ptycho_probe_exitwave": [_P, _c.c_int64, _P],
}
for _name, _args in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _c.c_int
    globals()[_name] = _f
lib.ptycho_last_error.argtypes = [_P]
lib.ptycho_last_error.restype = _c.c_char_p
ptycho_last_error = lib.ptycho_last_error

EXPORTED = sorted(list(_SIGS) + ["ptycho_last_error"])


def tile_geometry(height, width, rows, cols, halo):
    """[(ext, interior)] per tile from the library's host geometry (no GPU needed)."""
    out = np.zeros((rows * cols, 8), np.int32)
    st = lib.ptycho_tile_geometry(height, width, rows, cols, halo, out.ctypes.data)
    if st != 0:
        raise PtychoError(st, lib.ptycho_last_error(None).decode())
    return [(tuple(int(v) for v in r[:4]), tuple(int(v) for v in r[4:])) for r in out]


def appp_schedule(height, width, rows, cols, halo):
    """The library's APPP hop list (src, dst, y0, y1, x0, x1, add), global order (no GPU needed)."""
    cnt = ctypes.c_int32()
    st = lib.ptycho_appp_schedule(height, width, rows, cols, halo, None, 0, ctypes.byref(cnt))
    if st != 0:
        raise PtychoError(st, lib.ptycho_last_error(None).decode())
    out = np.zeros((cnt.value, 7), np.int32)
    st = lib.ptycho_appp_schedule(height, width, rows, cols, halo, out.ctypes.data, cnt.value, ctypes.byref(cnt))
    if st != 0:
        raise PtychoError(st, lib.ptycho_last_error(None).decode())
    return [tuple(int(v) for v in r) for r in out]


class PtychoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _ptr(a):
    """Device pointer of a torch tensor or host pointer of a contiguous numpy array."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def _on_device(a):
    return 0 if (a is None or isinstance(a, np.ndarray)) else int(a.is_cuda)


_KIND = {"f32": (np.float32, "float32"), "c64": (np.complex64, "complex64")}


def _check(a, kind, count, device, what):
    """Validate a buffer handed to the C ABI: dtype, C-contiguity, element count, and for CUDA
    tensors the context's device.  The library trusts sizes, so a wrong buffer would otherwise be
    read or written out of bounds (EARG instead)."""
    if a is None:
        return
    npt, tname = _KIND[kind]
    if isinstance(a, np.ndarray):
        ok_type, contig, numel = a.dtype == npt, a.flags["C_CONTIGUOUS"], a.size
    else:
        ok_type, contig, numel = str(a.dtype) == "torch." + tname, a.is_contiguous(), a.numel()
        if a.is_cuda and a.device.index != device:
            raise PtychoError(1, f"{what}: tensor on cuda:{a.device.index}, context on cuda:{device}")
    if not ok_type:
        raise PtychoError(1, f"{what}: dtype {a.dtype}, expected {tname}")
    if not contig:
        raise PtychoError(1, f"{what}: not C-contiguous")
    if count is not None and numel != count:
        raise PtychoError(1, f"{what}: {numel} elements, expected {count}")


class Ptycho:
    """One context = one rank's share of the reconstruction (ptycho_create ... ptycho_destroy)."""

    def __init__(self, n, slices, height, width, sigma=0.1, prop_c=3.135, alpha=1.0, alpha_acc=None,
                 tau=1e-4, pass_period=0, flags=0, device=0, stream=None):
        import torch
        self.torch = torch
        self.cfg = ptycho_config(n, slices, height, width, sigma, prop_c, alpha,
                                 alpha if alpha_acc is None else alpha_acc, tau, pass_period, flags)
        self.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        self.stream = stream
        h = _P()
        st = lib.ptycho_create(ctypes.byref(self.cfg), device, _P(stream), ctypes.byref(h))
        if st != 0:
            raise PtychoError(st, lib.ptycho_last_error(None).decode())
        self.h = h
        self.workspace = None

    def _ck(self, st):
        if st != 0:
            raise PtychoError(st, lib.ptycho_last_error(self.h).decode())

    def close(self):
        """Wait for every queued library kernel (tile, copy and context streams), then destroy the
        context, and only then release the workspace to PyTorch's caching allocator (a kernel still
        in flight must never see its memory handed to another tensor)."""
        if getattr(self, "h", None):
            lib.ptycho_synchronize(self.h)
            lib.ptycho_destroy(self.h)  # also synchronizes (and fences the P2P peers)
            self.h = None
        self.workspace = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        st = lib.ptycho_nccl_unique_id(buf, 128)
        if st != 0:
            raise PtychoError(st, lib.ptycho_last_error(None).decode())
        return buf.raw

    def set_tiles(self, rows, cols, halo, tile_owner=None, nccl_id=None, rank=0, nranks=1):
        own = None if tile_owner is None else np.ascontiguousarray(tile_owner, dtype=np.int32)
        nid = None if nccl_id is None else ctypes.create_string_buffer(bytes(nccl_id), 128)
        self._own = own
        self._ck(lib.ptycho_set_tiles(self.h, rows, cols, halo, _ptr(own), nid, rank, nranks))
        self.rows, self.cols = rows, cols

    def set_tiles_hve(self, rows, cols, halo, margin, tile_owner=None, nccl_id=None, rank=0, nranks=1):
        """Halo Voxel Exchange baseline: probes within `margin` px of a tile's interior
        are duplicated onto it; iterate = independent SGD sweeps + halo copy-paste."""
        own = None if tile_owner is None else np.ascontiguousarray(tile_owner, dtype=np.int32)
        nid = None if nccl_id is None else ctypes.create_string_buffer(bytes(nccl_id), 128)
        self._own = own
        self._ck(lib.ptycho_set_tiles_hve(self.h, rows, cols, halo, margin, _ptr(own), nid, rank, nranks))
        self.rows, self.cols = rows, cols

    def set_scan(self, centers):
        self._centers = np.ascontiguousarray(centers, dtype=np.int32)
        self._ck(lib.ptycho_set_scan(self.h, self._centers.ctypes.data, len(self._centers)))

    def local_probes(self):
        cnt = ctypes.c_int64()
        self._ck(lib.ptycho_local_probes(self.h, None, ctypes.byref(cnt)))
        ids = np.zeros(cnt.value, dtype=np.int64)
        self._ck(lib.ptycho_local_probes(self.h, ids.ctypes.data, ctypes.byref(cnt)))
        return ids

    def tile_probe_count(self, tile):
        cnt = ctypes.c_int64()
        self._ck(lib.ptycho_tile_probe_count(self.h, tile, ctypes.byref(cnt)))
        return cnt.value

    def tile_rect(self, tile):
        ext = np.zeros(4, np.int32)
        inter = np.zeros(4, np.int32)
        self._ck(lib.ptycho_tile_rect(self.h, tile, ext.ctypes.data, inter.ctypes.data))
        return tuple(int(v) for v in ext), tuple(int(v) for v in inter)

    def set_schedule(self, batched, max_batch=8):
        self._ck(lib.ptycho_set_schedule(self.h, int(bool(batched)), max_batch))

    def workspace_bytes(self):
        b = ctypes.c_size_t()
        self._ck(lib.ptycho_workspace_bytes(self.h, ctypes.byref(b)))
        return b.value

    def allocate_workspace(self):
        nbytes = self.workspace_bytes()
        self.workspace = self.torch.empty(nbytes + 256, dtype=self.torch.uint8, device=f"cuda:{self.device}")
        base = self.workspace.data_ptr()
        off = (-base) % 256
        self._ck(lib.ptycho_set_workspace(self.h, base + off, nbytes))
        return nbytes

    def set_probe(self, probe):
        if isinstance(probe, np.ndarray):
            probe = np.ascontiguousarray(probe, dtype=np.complex64)
        _check(probe, "c64", self.cfg.n ** 2, self.device, "probe")
        self._ck(lib.ptycho_set_probe(self.h, _ptr(probe), _on_device(probe)))

    def load_measurements(self, amp, first_local=0, flags=0):
        if isinstance(amp, np.ndarray):
            amp = np.ascontiguousarray(amp, dtype=np.float32)
        _check(amp, "f32", len(amp) * self.cfg.n ** 2, self.device, "measurements")
        self._ck(lib.ptycho_load_measurements(self.h, _ptr(amp), _on_device(amp), first_local, len(amp), flags))

    def read_measurements(self, first_local=0, count=None, out=None):
        if count is None:
            count = len(self.local_probes()) - first_local
        n = self.cfg.n
        if out is None:
            out = np.zeros((count, n, n), np.float32)
        _check(out, "f32", count * n * n, self.device, "read_measurements out")
        if not isinstance(out, np.ndarray) and out.is_cuda:
            raise PtychoError(1, "read_measurements writes host memory: pass a numpy array or a CPU tensor")
        self._ck(lib.ptycho_read_measurements(self.h, _ptr(out), first_local, count))
        return out

    def set_volume(self, volume=None):
        if isinstance(volume, np.ndarray):
            volume = np.ascontiguousarray(volume, dtype=np.float32)
        c = self.cfg
        _check(volume, "f32", c.slices * c.height * c.width, self.device, "volume")
        self._ck(lib.ptycho_set_volume(self.h, _ptr(volume), _on_device(volume)))

    def simulate_measurements(self):
        self._ck(lib.ptycho_simulate_measurements(self.h))

    def forward_grad(self, first, count, want_loss=False):
        loss = ctypes.c_double()
        self._ck(lib.ptycho_forward_grad(self.h, first, count, ctypes.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def appp_passes(self):
        self._ck(lib.ptycho_appp_passes(self.h))

    def set_appp_transport(self, mode):
        """PTYCHO_APPP_AUTO / _NCCL / _P2P (before the first APPP call)."""
        self._ck(lib.ptycho_set_appp_transport(self.h, mode))

    def appp_transport(self):
        v = ctypes.c_int32()
        self._ck(lib.ptycho_appp_transport(self.h, ctypes.byref(v)))
        return {0: "auto", 1: "nccl", 2: "p2p"}[v.value]

    def step(self):
        self._ck(lib.ptycho_step(self.h))

    def iterate(self, want_loss=False):
        loss = ctypes.c_double()
        self._ck(lib.ptycho_iterate(self.h, ctypes.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def stitch(self, out=None, root=0, rank=0):
        c = self.cfg
        if out is None and rank == root:
            out = np.zeros((c.slices, c.height, c.width), np.float32)
        _check(out, "f32", c.slices * c.height * c.width, self.device, "stitch out")
        self._ck(lib.ptycho_stitch(self.h, _ptr(out), _on_device(out), root))
        return out

    def synchronize(self):
        self._ck(lib.ptycho_synchronize(self.h))

    def kernel_launches(self):
        v = ctypes.c_int64()
        self._ck(lib.ptycho_kernel_launches(self.h, ctypes.byref(v)))
        return v.value

    PASS_KINDS = ["fwd_first_prop", "fwd_first_fft", "fwd_mid", "fwd_last", "turn", "simulate",
                  "bwd_last_prop", "bwd_last_end", "bwd_mid", "bwd_end", "exit_complete",
                  "recon_first", "recon_mid", "recon_end"]

    def profile_chain(self, tile, first, count):
        ms = np.zeros(len(self.PASS_KINDS), np.float64)
        cnt = np.zeros(len(self.PASS_KINDS), np.int64)
        self._ck(lib.ptycho_profile_chain(self.h, tile, first, count, ms.ctypes.data, cnt.ctypes.data))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(self.PASS_KINDS) if cnt[i]}

    def profile_iteration(self):
        """One real iteration with serial phases; per-phase ms on this rank (collective)."""
        ms = np.zeros(8, np.float64)
        self._ck(lib.ptycho_profile_iteration(self.h, ms.ctypes.data))
        d = dict(zip(["total_ms", "compute_ms", "wait_ms", "comm_ms", "acc_step_ms", "sender_hold_ms",
                      "nvlink_copy_ms", "nvlink_copy_bytes"], (float(v) for v in ms)))
        d["nvlink_copy_gbs"] = d["nvlink_copy_bytes"] / (d["nvlink_copy_ms"] * 1e6) if d["nvlink_copy_ms"] > 0 else None
        return d

    def debug_errors(self):
        """(error bits, checks_built) of the PTYCHO_DEBUG_CHECKS ordering checks (clears the bits)."""
        bits = ctypes.c_uint32()
        built = ctypes.c_int32()
        self._ck(lib.ptycho_debug_errors(self.h, ctypes.byref(bits), ctypes.byref(built)))
        return bits.value, bool(built.value)

    # ---- debug exports
    def debug_read_tile(self, tile, which):
        ext, _ = self.tile_rect(tile)
        out = np.zeros((self.cfg.slices, ext[2] - ext[0], ext[3] - ext[1]), np.float32)
        self._ck(lib.ptycho_debug_read_tile(self.h, tile, which, out.ctypes.data))
        return out

    def debug_write_tile(self, tile, which, arr):
        arr = np.ascontiguousarray(arr, dtype=np.float32)
        self._ck(lib.ptycho_debug_write_tile(self.h, tile, which, arr.ctypes.data))

    def debug_probe_grad(self, tile, probe):
        n, s = self.cfg.n, self.cfg.slices
        g = np.zeros((s, n, n), np.float32)
        loss = ctypes.c_double()
        self._ck(lib.ptycho_debug_probe_grad(self.h, tile, probe, g.ctypes.data, ctypes.byref(loss)))
        return g, loss.value

    def debug_exit_wave(self, tile, probe):
        n = self.cfg.n
        psi = np.zeros((n, n), np.complex64)
        self._ck(lib.ptycho_debug_exit_wave(self.h, tile, probe, psi.ctypes.data))
        return psi

    def probe_grad(self, probe, out=None):
        """d f_i / d V over the full window of GLOBAL probe `probe` (host numpy or device tensor out)."""
        n, s = self.cfg.n, self.cfg.slices
        g = np.zeros((s, n, n), np.float32) if out is None else out
        _check(g, "f32", s * n * n, self.device, "probe_grad out")
        loss = ctypes.c_double()
        self._ck(lib.ptycho_probe_grad(self.h, probe, _ptr(g), ctypes.byref(loss)))
        return g, loss.value

    def probe_exitwave(self, probe, out=None):
        n = self.cfg.n
        psi = np.zeros((n, n), np.complex64) if out is None else out
        _check(psi, "c64", n * n, self.device, "probe_exitwave out")
        self._ck(lib.ptycho_probe_exitwave(self.h, probe, _ptr(psi)))
        return psi
