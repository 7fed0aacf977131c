"""stl -- GPU ingestion of ASCII STL: drop-in for the
reference's ``geometry.parse_stl(data, weld_tol=None)`` (geometry.py:128-209)
with its ``_weld`` (geometry.py:212-225) and TriangleMesh normals
(geometry.py:114-124).

The text goes to HBM once; tokenizing, the grammar check, the decimal ->
double conversion (correctly rounded, bit-identical to Python float()), the
vertex weld and the normals run in csrc/vf_stl.cu.  The host only reads back
the counts, the extent (for the default weld tolerance) and, on error, one
token to compose the reference's StlParseError message.  The result is a
TriangleMesh (host arrays, as the reference returns) that already carries its
packed device face records, so embedding it needs no second upload.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Union

import numpy as np

from . import _lib
from .datatypes import DeviceMesh
from .errors import MeshError, StlParseError
from .mesh import TriangleMesh

_WORDS = ["solid", "facet", "normal", "outer", "loop", "vertex", "endloop", "endfacet", "endsolid"]
# facet slot -> (kind, vertex) for the error context: 'k' keyword, 'n' normal, 'v' vertex j
_SLOTS = (["k", "k", "n", "n", "n", "k", "k", "k"] + ["v1"] * 3 + ["k"] + ["v2"] * 3 + ["k"]
          + ["v3"] * 3 + ["k", "k"])
_SLOTS = ["k", "k", "n", "n", "n", "k", "k", "k", "v1", "v1", "v1", "k", "v2", "v2", "v2", "k",
          "v3", "v3", "v3", "k", "k"]


def _line_of(text: str, off: int) -> int:
    # the reference numbers tokens by text.splitlines(), starting at 1
    return len((text[:off] + "x").splitlines())


def _token(text: str, off: int) -> str:
    return text[off:].split(maxsplit=1)[0]


def _message(text: str, info, off: int) -> str:
    kind, t, word, head, n_tok = info[1], info[2], info[3], info[4], info[5]
    n_facets = info[0]
    if t == 0 or (word == 0 and kind in (1, 3) and t < head):
        ctx = "header"
    elif word == 8:
        ctx = f"trailer after facet {n_facets}"
    else:
        k = (t - head) // 21
        slot = (t - head) % 21
        ctx = f"facet {k + 1}"
        s = _SLOTS[slot]
        if s == "n":
            ctx += " normal"
        elif s.startswith("v"):
            ctx += f" vertex {s[1]}"
    if kind == 3:
        return f"unexpected end of file while reading {ctx}"
    ln, tok = _line_of(text, off), _token(text, off)
    if kind == 1:
        return f"line {ln}: expected '{_WORDS[word]}' in {ctx}, got '{tok}'"
    return f"line {ln}: bad number '{tok}' in {ctx}"


def _ascii_canonical(text: str):
    """A str input with non-ASCII characters (geometry.py:138-149 parses a
    str without the ASCII check) as an equivalent ASCII stream: the
    reference's own line split (str.splitlines) and token split (str.split,
    Unicode whitespace included), one line per line so line numbers stay.
    Non-ASCII tokens become a number's repr when float() accepts them, else a
    unique ASCII placeholder that error messages map back."""
    lines, subst = [], {}
    for line in text.splitlines():
        toks = []
        for tok in line.split():
            if not tok.isascii():
                try:
                    tok = repr(float(tok))
                except ValueError:
                    key = f"@u{len(subst)}@"
                    subst[key] = tok
                    tok = key
            toks.append(tok)
        lines.append(" ".join(toks))
    return "\n".join(lines), subst


def parse_stl(data: Union[bytes, str], weld_tol: Optional[float] = None,
              stream=None) -> TriangleMesh:
    """geometry.parse_stl on the GPU.  Same result arrays (bit-identical) and
    the same StlParseError / MeshError conditions and messages."""
    import torch
    lib = _lib.require_cuda()
    subst = {}
    if isinstance(data, str) and not data.isascii():
        data, subst = _ascii_canonical(data)
    raw = data.encode("ascii") if isinstance(data, str) else bytes(data)
    n = len(raw)
    st = _lib.stream_ptr(stream)
    # one pageable H2D copy of the text (no host-side copy / pinning of the bytes)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # read-only buffer: only read by the copy
        host = torch.from_numpy(np.frombuffer(raw, dtype=np.uint8)) if n else torch.zeros(1, dtype=torch.uint8)
        d_text = host.to("cuda")
    ws = torch.empty(int(lib.vf_stl_workspace_size(n)), dtype=torch.uint8, device="cuda")
    info = (C.c_int64 * 6)()
    ext = (C.c_double * 6)()
    off = C.c_int64(-1)
    _lib.check(lib.vf_stl_scan(_lib.ptr(d_text), n, _lib.ptr(ws), ws.numel(), info, ext, C.byref(off), st),
               "parse_stl")
    info = list(info)
    if info[1] == 4:  # bytes input only: a str is canonicalised to ASCII above
        raise StlParseError("not an ASCII STL stream")
    text = raw.decode("ascii") if info[1] else ""
    if info[1]:
        msg = _message(text, info, int(off.value))
        for k, v in subst.items():
            msg = msg.replace(k, v)
        raise StlParseError(msg)
    nf = int(info[0])
    if nf == 0:
        raise StlParseError("empty mesh: STL contains zero facets")
    lo, hi = np.array(ext[:3]), np.array(ext[3:])
    with np.errstate(over="ignore"):  # as the reference: an infinite extent stays inf
        extent = float((hi - lo).max()) or 1.0
    tol = weld_tol if weld_tol is not None else 1e-12 * extent
    weld = torch.empty(int(lib.vf_stl_weld_workspace_size(nf)), dtype=torch.uint8, device="cuda")
    verts = torch.empty((3 * nf, 3), dtype=torch.float64, device="cuda")
    faces = torch.empty((nf, 3), dtype=torch.int64, device="cuda")
    fc = torch.empty((nf, 9), dtype=torch.float64, device="cuda")
    nrm = torch.empty((nf, 3), dtype=torch.float64, device="cuda")
    packed = torch.empty((nf, 12), dtype=torch.float64, device="cuda")
    nv, degen = C.c_int64(0), C.c_int32(0)
    _lib.check(lib.vf_stl_build(_lib.ptr(d_text), n, _lib.ptr(ws), ws.numel(), nf, float(tol), _lib.ptr(weld),
                                weld.numel(), _lib.ptr(verts), _lib.ptr(faces), _lib.ptr(fc), _lib.ptr(nrm),
                                _lib.ptr(packed), C.byref(nv), C.byref(degen), st), "parse_stl")
    if degen.value:
        raise MeshError("degenerate face (zero normal)")
    v = fc.view(nf, 3, 3)
    area = float(0.5 * torch.linalg.norm(torch.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0], dim=1), dim=1).sum())
    mesh = TriangleMesh.from_arrays(verts[:nv.value].cpu().numpy(), faces.cpu().numpy(), fc.cpu().numpy(),
                                    nrm.cpu().numpy())
    mesh._vf_device_mesh = DeviceMesh(packed, nf, area)
    return mesh
