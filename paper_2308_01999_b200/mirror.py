"""Host mirrors of device segments that notice writes.

The reference hands out its amplitude array itself (statevec.py:126), so
callers mutate it in place (`sv.amplitudes[:] = amps`, reference
tests/test_circuits.py:79).  Here the array is a host copy of HBM; a write
must be re-uploaded before the next device operation, but a read must not
(re-uploading a 64 GiB mirror because someone looked at it costs seconds).

`MirrorArray` is an ndarray subclass whose mutating entry points —
subscript assignment, in-place ufuncs (`a *= 2`, `np.add(x, y, out=a)`),
the mutating NumPy functions (`np.copyto`, `np.put`, `np.place`,
`np.putmask`, `np.fill_diagonal`) and the mutating methods (`fill`, `sort`,
`put`, `partition`, `itemset`, `setfield`, `byteswap(inplace)`) — flag the
owning state dirty.  Views (slices, reshapes) keep the owner, so writes
through them are seen too.  Writes through raw buffers (ctypes pointers,
memoryviews) are not; call the owner's ``mark_host_dirty()`` after those.
"""

from __future__ import annotations

import numpy as np

_MUTATING_FUNCS = {np.copyto, np.put, np.place, np.putmask, np.fill_diagonal}


class MirrorArray(np.ndarray):
    _owner = None  # callable invoked on the first write

    def __array_finalize__(self, obj):
        # views keep the owner (writes through them reach the state); copies
        # (copy(), astype(), fancy-index reads) own their memory and do not
        self._owner = getattr(obj, "_owner", None) if self.base is not None else None

    def _touch(self):
        cb = self._owner
        if cb is not None:
            cb()

    def __setitem__(self, key, value):
        self._touch()
        super().__setitem__(key, value)

    def __array_ufunc__(self, ufunc, method, *inputs, out=None, **kwargs):
        if out is not None:
            for o in out:
                if isinstance(o, MirrorArray):
                    o._touch()
            kwargs["out"] = tuple(o.view(np.ndarray) if isinstance(o, MirrorArray) else o for o in out)
        args = [x.view(np.ndarray) if isinstance(x, MirrorArray) else x for x in inputs]
        res = getattr(ufunc, method)(*args, **kwargs)
        if out is not None:  # in-place (`a *= 2`): the caller keeps the mirror object
            return out[0] if len(out) == 1 else out
        # computed values are plain arrays: they are not views of the state
        return res

    def __array_function__(self, func, types, args, kwargs):
        if func in _MUTATING_FUNCS and args and isinstance(args[0], MirrorArray):
            args[0]._touch()
        return super().__array_function__(func, tuple(np.ndarray if issubclass(t, MirrorArray) else t
                                                      for t in types), args, kwargs)

    # mutating methods
    def fill(self, value):
        self._touch()
        super().fill(value)

    def sort(self, *a, **k):
        self._touch()
        super().sort(*a, **k)

    def put(self, *a, **k):
        self._touch()
        super().put(*a, **k)

    def partition(self, *a, **k):
        self._touch()
        super().partition(*a, **k)

    def itemset(self, *a):  # NumPy < 2
        self._touch()
        return super().itemset(*a)

    def setfield(self, *a, **k):
        self._touch()
        return super().setfield(*a, **k)

    def byteswap(self, inplace=False):
        if inplace:
            self._touch()
        return super().byteswap(inplace)


def mirror_of(buf: np.ndarray, on_write) -> MirrorArray:
    """A MirrorArray view of `buf` whose writes call `on_write()`."""
    m = buf.view(MirrorArray)
    m._owner = on_write
    return m
