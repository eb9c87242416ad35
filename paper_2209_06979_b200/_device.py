"""Host <-> device plumbing for the C ABI (torch is used for memory and streams only).

Containers may hold numpy arrays (host) or torch tensors. Device copies of
host arrays are cached on the (immutable) container object, so repeated calls
with the same sparse matrix pay the host-to-device copy once.
"""

from __future__ import annotations

import warnings

import numpy as np

from . import _native as N


def torch():
    import torch as _t
    return _t


def is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def on_device(x) -> bool:
    return is_torch(x) and x.is_cuda


def to_dev(x, np_dtype, device=None):
    """numpy / torch -> contiguous CUDA tensor with the byte layout of np_dtype."""
    t = torch()
    if is_torch(x):
        tt = x
    else:
        arr = np.ascontiguousarray(np.asarray(x, dtype=np_dtype))
        view = {np.uint32: np.int32, np.uint64: np.int64}.get(np.dtype(np_dtype).type, None)
        if view is not None:
            arr = arr.view(view)
        with warnings.catch_warnings():  # read-only (frozen) host arrays: copied to the device below
            warnings.simplefilter("ignore", UserWarning)
            tt = t.from_numpy(arr)
    dev = device if device is not None else t.device("cuda", t.cuda.current_device())
    return tt.to(dev, non_blocking=True).contiguous()


def _freeze(obj):
    """Make the container's host arrays read-only once a device copy of them is cached:
    the containers are immutable by contract (frozen dataclasses, as in the reference),
    and an in-place edit would otherwise leave the cached device copy stale."""
    for name in ("row_begin", "row_end", "row_offsets", "col_indices", "words", "values"):
        x = obj.__dict__.get(name)
        x = getattr(x, "words", x)
        if isinstance(x, np.ndarray) and x.flags.writeable:
            try:
                x.flags.writeable = False
            except ValueError:
                pass


def cached(obj, key, make):
    _freeze(obj)
    cache = obj.__dict__.get("_dev_cache")
    if cache is None:
        cache = {}
        object.__setattr__(obj, "_dev_cache", cache)
    t = torch()
    dkey = (key, t.cuda.current_device())
    if dkey not in cache:
        cache[dkey] = make()
    return cache[dkey]


def words_of(values):
    """Packed words (PackedArray / PackedMatrix) or a raw 32-bit array -> device int32."""
    w = getattr(values, "words", values)
    if is_torch(w):
        return w.cuda().contiguous().view(torch().int32) if w.element_size() == 4 else w.cuda().contiguous()
    arr = np.asarray(w)
    if arr.dtype.itemsize != 4:
        raise ValueError("expected 32-bit words")
    return to_dev(arr.view(np.int32), np.int32)


def any_host(*objs) -> bool:
    """True when any container field is a host (numpy) array -> return numpy outputs."""
    for o in objs:
        w = getattr(o, "words", None)
        if w is None:
            w = getattr(getattr(o, "values", None), "words", getattr(o, "values", None))
        if w is not None and not on_device(w):
            return True
    return False


def srbcrs_struct(m):
    def make():
        begin = to_dev(m.row_begin, np.int64)
        end = to_dev(m.row_end, np.int64)
        idx = to_dev(m.col_indices, np.uint32)
        words = words_of(m.values)
        bits = getattr(m.values, "bit_width", 32)
        s = N.McSrBcrs(m.scalar_rows, m.scalar_cols, m.vector_length, m.stride, bits,
                       int(bool(m.shuffled)), int(idx.numel()), N.ptr(begin), N.ptr(end),
                       N.ptr(idx), N.ptr(words))
        return s, (begin, end, idx, words)
    return cached(m, "srbcrs", make)


def dense_struct(pm):
    from .qint import ROW_MAJOR

    def make():
        words = words_of(pm)
        layout = N.MC_ROW_MAJOR if pm.layout == ROW_MAJOR else N.MC_COL_MAJOR
        return N.McDense(pm.rows, pm.cols, pm.bit_width, layout, N.ptr(words)), (words,)
    return cached(pm, "dense", make)


def bcrs_struct(b):
    def make():
        offs = to_dev(b.row_offsets, np.int64)
        idx = to_dev(b.col_indices, np.uint32)
        s = N.McBcrs(b.scalar_rows, b.scalar_cols, b.vector_length, 0, int(idx.numel()),
                     N.ptr(offs), N.ptr(idx))
        return s, (offs, idx)
    return cached(b, "bcrs", make)


_status = {}


def status_word():
    """Per-device status word (uint32) handed to kernels for data-dependent errors."""
    t = torch()
    dev = t.cuda.current_device()
    if dev not in _status:
        _status[dev] = t.zeros(1, dtype=t.int32, device=f"cuda:{dev}")
    return _status[dev]


def fresh_status():
    """A zeroed status word for one checked launch: flags left by unchecked launches
    (status_word) or by launches on other streams never reach a checked call."""
    t = torch()
    return t.zeros(1, dtype=t.int32, device=f"cuda:{t.cuda.current_device()}")


def fetch_status(status, stream=None):
    N.check(N.lib().mc_status_fetch(N.ptr(status), N.stream_ptr(stream)))
