"""Device-resident model and nonzeros, plus thin wrappers over libsptk.

PyTorch is used only to own device memory and to supply the current stream;
all arithmetic happens in the sm_100a kernels behind include/sptk.h.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import check, f64arr, i64arr, ptr, stream_ptr


def _torch():
    import torch

    return torch


def record_words(order: int, f64: bool) -> int:
    return int(_lib.load().sptk_record_words(order, 1 if f64 else 0))


class DeviceModel:
    """Packed A(n)/B(n) on the device in the reference's layout
    (trainer.py:135-141, _loops.py:8-10), fp32 (throughput) or fp64
    (verification)."""

    def __init__(self, model, f64: bool = False, device=None, pad_rank: int | None = None):
        """pad_rank = P zero-pads every J_n and R up to P on the device.  The
        padded model is exactly equivalent (padded rows/columns of A and B are
        zero and every gradient on them is zero), so ranks below the smallest
        tensor-core tile (J = R = 4 -> 8) run on the tcgen05 kernels;
        ``download_into`` strips the padding."""
        torch = _torch()
        _lib.require_cuda()
        self.device = torch.device(device or "cuda")
        self.f64 = f64
        self.dtype = torch.float64 if f64 else torch.float32
        self.order = model.order
        self.dims = tuple(model.dims)
        self.true_jr = [int(j) for j in model.j_ranks]
        self.true_r = int(model.r_core)
        P = int(pad_rank) if pad_rank else 0
        self.rcore = max(self.true_r, P)
        self.jr = np.asarray([max(j, P) for j in self.true_jr], dtype=np.int64)
        sizes_a = [d * j for d, j in zip(model.dims, self.jr)]
        sizes_b = [int(j) * self.rcore for j in self.jr]
        self.foff = np.concatenate([[0], np.cumsum(sizes_a)]).astype(np.int64)
        self.coff = np.concatenate([[0], np.cumsum(sizes_b)]).astype(np.int64)
        npdt = np.float64 if f64 else np.float32

        def padded(m, rows, cols):
            m = np.asarray(m, dtype=np.float64)
            if m.shape == (rows, cols):
                return m.ravel()
            out = np.zeros((rows, cols))
            out[: m.shape[0], : m.shape[1]] = m
            return out.ravel()

        # packed straight into one host buffer of the device dtype, one upload
        fac = np.empty(int(self.foff[-1]), dtype=npdt)
        for n, (a, j) in enumerate(zip(model.factors, self.jr)):
            dst = fac[int(self.foff[n]): int(self.foff[n + 1])].reshape(a.shape[0], int(j))
            if a.shape[1] == int(j):
                np.copyto(dst, a, casting="unsafe")
            else:
                dst[:] = 0
                np.copyto(dst[:, : a.shape[1]], a, casting="unsafe")
        cor = np.concatenate([padded(b, int(j), self.rcore) for b, j in zip(model.core_factors, self.jr)]).astype(npdt)
        self.fac = torch.from_numpy(fac).to(self.device)
        self.cor = torch.from_numpy(cor).to(self.device)
        self.cor_size = int(self.coff[-1])
        # ctypes views of the small host arrays (kept alive on self)
        self._foff, self.p_foff = i64arr(self.foff)
        self._coff, self.p_coff = i64arr(self.coff)
        self._jr, self.p_jr = i64arr(self.jr)

    def download_into(self, model) -> None:
        # device dtype over the bus (fp32: half the bytes), widened by copyto
        fac = self.fac.cpu().numpy()
        cor = self.cor.cpu().numpy()
        for n, a in enumerate(model.factors):
            full = fac[self.foff[n]: self.foff[n + 1]].reshape(a.shape[0], int(self.jr[n]))
            np.copyto(a, full[:, : a.shape[1]])
        for n, b in enumerate(model.core_factors):
            full = cor[self.coff[n]: self.coff[n + 1]].reshape(int(self.jr[n]), self.rcore)
            np.copyto(b, full[: b.shape[0], : b.shape[1]])


class DeviceCoo:
    """Nonzeros as packed device records {i_0..i_{N-1}, value} in source order."""

    def __init__(self, indices: np.ndarray, values: np.ndarray, f64: bool = False, device=None):
        torch = _torch()
        _lib.require_cuda()
        dev = torch.device(device or "cuda")
        idx = np.ascontiguousarray(indices, dtype=np.int64)
        self.nnz = int(idx.shape[0])
        self.order = int(idx.shape[1])
        self.f64 = f64
        self.rw = record_words(self.order, f64)
        self.rec = torch.empty(max(self.nnz, 1) * self.rw, dtype=torch.int32, device=dev)
        vals = np.ascontiguousarray(values, dtype=np.float64)
        if self.nnz and not f64 and dev.index in (None, torch.cuda.current_device()):
            # fp32 records packed by the upload threads (sptk_h2d_pack)
            torch.cuda.current_stream().synchronize()
            check(_lib.load().sptk_h2d_pack(ptr(self.rec), idx.ctypes.data, vals.ctypes.data, self.nnz, self.order, 0),
                  "sptk_h2d_pack")
        elif self.nnz:
            d_idx = torch.from_numpy(idx).to(dev)
            d_val = torch.from_numpy(vals).to(dev)
            check(_lib.load().sptk_pack_records(ptr(d_idx), ptr(d_val), self.nnz, self.order,
                                                1 if f64 else 0, ptr(self.rec), stream_ptr()),
                  "sptk_pack_records")
            del d_idx, d_val


def eval_sums(dm: DeviceModel, coo: DeviceCoo, sums=None):
    """Launch K6 and return the device (2,) fp64 tensor {sum sq, sum abs}."""
    torch = _torch()
    L = _lib.load()
    if sums is None:
        sums = torch.zeros(2, dtype=torch.float64, device=dm.fac.device)
    fn = L.sptk_eval_f64 if dm.f64 else L.sptk_eval
    check(fn(ptr(coo.rec), coo.rw, coo.nnz, ptr(dm.fac), dm.p_foff, ptr(dm.cor), dm.p_coff, dm.p_jr,
             dm.order, dm.rcore, None, ptr(sums), stream_ptr()), "sptk_eval")
    return sums


def rmse_mae_device(dm: DeviceModel, coo: DeviceCoo):
    if coo.nnz == 0:
        raise ValueError("dataset is empty")
    s = eval_sums(dm, coo).cpu().numpy()
    return float(np.sqrt(s[0] / coo.nnz)), float(s[1] / coo.nnz)


def predict_device(model, indices: np.ndarray) -> np.ndarray:
    torch = _torch()
    dm = DeviceModel(model)
    m = indices.shape[0]
    coo = DeviceCoo(indices, np.zeros(m), f64=False)
    out = torch.empty(max(m, 1), dtype=torch.float32, device=dm.fac.device)
    L = _lib.load()
    check(L.sptk_eval(ptr(coo.rec), coo.rw, m, ptr(dm.fac), dm.p_foff, ptr(dm.cor), dm.p_coff, dm.p_jr,
                      dm.order, dm.rcore, ptr(out), None, stream_ptr()), "sptk_eval")
    return out[:m].double().cpu().numpy()


def predict_device_f64(model, indices: np.ndarray) -> np.ndarray:
    """fp64 device evaluation (used for data synthesis at scale)."""
    torch = _torch()
    dm = DeviceModel(model, f64=True)
    m = indices.shape[0]
    coo = DeviceCoo(indices, np.zeros(m), f64=True)
    out = torch.empty(max(m, 1), dtype=torch.float64, device=dm.fac.device)
    check(_lib.load().sptk_eval_f64(ptr(coo.rec), coo.rw, m, ptr(dm.fac), dm.p_foff, ptr(dm.cor), dm.p_coff,
                                    dm.p_jr, dm.order, dm.rcore, ptr(out), None, stream_ptr()), "sptk_eval_f64")
    return out[:m].cpu().numpy()


class SharedBuffer:
    """Device memory another process (or GPU) can map: cudaMalloc'd by libsptk
    (sptk_shared_alloc) so its CUDA IPC handle covers exactly this buffer.
    ``view`` returns zero-copy torch tensors over it.  Freed by ``close``."""

    _TYPESTR = {"float32": "<f4", "int32": "<i4", "float64": "<f8", "int64": "<i8", "uint8": "|u1"}

    def __init__(self, nbytes: int):
        import ctypes

        p = ctypes.c_void_p()
        check(_lib.load().sptk_shared_alloc(int(nbytes), ctypes.byref(p)), "sptk_shared_alloc")
        self.ptr = int(p.value)
        self.nbytes = int(nbytes)

    def view(self, dtype, numel: int, offset: int = 0):
        torch = _torch()
        name = str(dtype).replace("torch.", "")

        class _Cai:
            pass

        o = _Cai()
        o.__cuda_array_interface__ = {"shape": (int(numel),), "typestr": self._TYPESTR[name],
                                      "data": (self.ptr + int(offset), False), "version": 3, "strides": None}
        return torch.as_tensor(o, device="cuda")

    def ipc_handle(self) -> bytes:
        import ctypes

        buf = ctypes.create_string_buffer(64)
        check(_lib.load().sptk_ipc_get(self.ptr, buf), "sptk_ipc_get")
        return buf.raw

    def close(self) -> None:
        if self.ptr:
            check(_lib.load().sptk_shared_free(self.ptr), "sptk_shared_free")
            self.ptr = 0


def ipc_open(handle: bytes) -> int:
    """Map a peer's SharedBuffer (its ipc_handle()); returns the device address."""
    import ctypes

    p = ctypes.c_void_p()
    check(_lib.load().sptk_ipc_open(bytes(handle), ctypes.byref(p)), "sptk_ipc_open")
    return int(p.value)
