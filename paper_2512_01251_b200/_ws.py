"""Device workspace cache: CUB-style two-phase workspaces are allocated once
per (purpose, size class) through PyTorch's caching allocator and reused."""
from __future__ import annotations

_cache = {}


def get(key: str, nbytes: int):
    import torch
    nbytes = max(int(nbytes), 256)
    buf = _cache.get(key)
    if buf is None or buf.numel() < nbytes:
        _cache.pop(key, None)
        buf = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        _cache[key] = buf
    return buf


def clear():
    _cache.clear()
