"""Problem files.

Two on-disk forms of a ``ProblemData``:

* **QOCOPROB 1** -- the reference's line-oriented text format
  (pkg/src/qsocp/fileio.py:1-122), same layout, so files written by either
  side load on the other.  One text line per nonzero: fine for desk-size
  problems, unusable at 10^8 nonzeros (the reference writes it with a Python
  loop per entry, fileio.py:34-44; here the columns are formatted by NumPy).
* **QOCOPROB 2** -- binary: a JSON header followed by the raw little-endian
  int64 / float64 arrays of the CSC matrices and vectors, each 64-byte aligned.
  ``load_problem(path)`` maps the file (``np.memmap``): nothing is parsed or
  copied, ``qs_setup`` reads the arrays straight out of the page cache, and
  ``pin=True`` page-locks the mapping (``qs_host_register``) so the host ->
  device copies run at full PCIe/C2C speed.  An optional fill-reducing
  permutation and free-form metadata (generator, seed, ...) travel in the same
  file, so an instance solved offline by the CPU oracle and on the GPU box is
  guaranteed to be the same bytes.

``save_problem`` / ``load_problem`` pick the form from the file's first bytes
(load) or from ``binary=`` / the ``.qp2`` suffix (save).
"""

from __future__ import annotations

import io
import json
import os

import numpy as np

from .errors import BadSparseStructure
from .problem import ConeSpec, ProblemData, validate_problem
from .sparse import SparseMatrixCSC, csc_from_triplets

MAGIC = "QOCOPROB"  # fileio.py:25
VERSION = 1  # fileio.py:26
BINARY_VERSION = 2
_ALIGN = 64
_HEADER_BYTES = 4096  # header block (magic line + JSON), padded; grows in 4 KiB steps if the metadata is large


# ------------------------------------------------------------------ text form
def _fmt_values(v) -> list:
    return [f"{float(x):.16e}" for x in v]  # fileio.py:29-30: 17 significant digits round-trip a float64


def problem_to_text(data: ProblemData) -> str:  # fileio.py:47-59
    cone = data.cone
    out = io.StringIO()
    out.write(f"{MAGIC} {VERSION}\n{data.n} {data.m} {data.p} {cone.orthant_dim} {cone.soc_count}\n")
    out.write(" ".join(str(int(q)) for q in cone.soc_dims) + "\n")
    for name, M in (("P", data.P), ("A", data.A), ("G", data.G)):
        out.write(f"MAT {name} {M.rows} {M.cols} {M.nnz}\n")
        if M.nnz:
            cols = M.column_of_entry()
            vals = _fmt_values(M.values)
            out.write("\n".join(f"{int(r)} {int(c)} {v}" for r, c, v in zip(M.row_indices, cols, vals)) + "\n")
    for name, v in (("c", data.c), ("b", data.b), ("h", data.h)):
        out.write(f"VEC {name} {len(v)}\n")
        if len(v):
            out.write("\n".join(_fmt_values(v)) + "\n")
    return out.getvalue()


class _Lines:
    def __init__(self, text: str):
        self.lines = text.splitlines()
        self.pos = 0

    def take(self, count=1):
        if self.pos + count > len(self.lines):
            raise BadSparseStructure("unexpected end of problem file")  # fileio.py:73-74
        chunk = self.lines[self.pos:self.pos + count]
        self.pos += count
        return chunk


def _read_matrix(rd: _Lines, name: str) -> SparseMatrixCSC:  # fileio.py:80-91
    head = rd.take()[0].split()
    if len(head) != 5 or head[0] != "MAT" or head[1] != name:
        raise BadSparseStructure(f"expected 'MAT {name} ...' header, got {head!r}")
    rows, cols, nnz = int(head[2]), int(head[3]), int(head[4])
    if nnz == 0:
        return csc_from_triplets(rows, cols, (np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)))
    try:
        body = np.array([ln.split() for ln in rd.take(nnz)])
        r, c, v = body[:, 0].astype(np.int64), body[:, 1].astype(np.int64), body[:, 2].astype(np.float64)
    except (ValueError, IndexError) as e:
        raise BadSparseStructure(f"malformed entry in matrix {name}: {e}") from None
    return csc_from_triplets(rows, cols, (r, c, v))


def _read_vector(rd: _Lines, name: str) -> np.ndarray:  # fileio.py:94-99
    head = rd.take()[0].split()
    if len(head) != 3 or head[0] != "VEC" or head[1] != name:
        raise BadSparseStructure(f"expected 'VEC {name} ...' header, got {head!r}")
    try:
        return np.array([float(t) for t in rd.take(int(head[2]))])
    except ValueError as e:
        raise BadSparseStructure(f"malformed entry in vector {name}: {e}") from None


def problem_from_text(text: str) -> ProblemData:  # fileio.py:102-117
    rd = _Lines(text)
    head = rd.take()[0].split()
    if head != [MAGIC, str(VERSION)]:
        raise BadSparseStructure(f"unsupported problem file header: {head!r}")
    n, m, p, l, nsoc = (int(t) for t in rd.take()[0].split())
    qline = rd.take()[0].split()
    if len(qline) != nsoc:
        raise BadSparseStructure(f"expected {nsoc} cone sizes, got {len(qline)}")
    cone = ConeSpec(l, tuple(int(q) for q in qline))
    P, A, G = _read_matrix(rd, "P"), _read_matrix(rd, "A"), _read_matrix(rd, "G")
    c, b, h = _read_vector(rd, "c"), _read_vector(rd, "b"), _read_vector(rd, "h")
    return validate_problem(ProblemData(n, m, p, P, c, A, b, G, h, cone))


# ---------------------------------------------------------------- binary form
_ARRAYS = (("soc_dims", np.int64), ("P_p", np.int64), ("P_i", np.int64), ("P_x", np.float64),
           ("A_p", np.int64), ("A_i", np.int64), ("A_x", np.float64),
           ("G_p", np.int64), ("G_i", np.int64), ("G_x", np.float64),
           ("c", np.float64), ("b", np.float64), ("h", np.float64), ("perm", np.int64))


def _arrays_of(data: ProblemData, perm):
    out = {"soc_dims": np.asarray(data.cone.soc_dims, np.int64), "c": data.c, "b": data.b, "h": data.h}
    for k, M in (("P", data.P), ("A", data.A), ("G", data.G)):
        out[k + "_p"], out[k + "_i"], out[k + "_x"] = M.col_pointers, M.row_indices, M.values
    if perm is not None:
        out["perm"] = np.asarray(perm, np.int64)
    return out


def save_problem_binary(data: ProblemData, path, perm=None, meta: dict | None = None) -> None:
    """Write QOCOPROB 2.  ``perm`` (optional): a fill-reducing permutation of the KKT system to ship with the
    problem; ``meta``: any JSON-serialisable description (generator name, seed, ...)."""
    arrs = _arrays_of(data, perm)
    header_bytes = _HEADER_BYTES
    while True:
        off = header_bytes
        table = {}
        for name, dt in _ARRAYS:
            if name not in arrs:
                continue
            a = np.ascontiguousarray(arrs[name], dtype=dt)
            table[name] = {"dtype": np.dtype(dt).str, "count": int(a.size), "offset": off}
            off += (a.nbytes + _ALIGN - 1) // _ALIGN * _ALIGN
        head = {"n": data.n, "m": data.m, "p": data.p, "l": data.cone.orthant_dim, "nsoc": data.cone.soc_count,
                "shapes": {k: [getattr(data, k).rows, getattr(data, k).cols] for k in "PAG"},
                "arrays": table, "meta": meta or {}}
        blob = (f"{MAGIC} {BINARY_VERSION}\n" + json.dumps(head) + "\n").encode()
        if len(blob) <= header_bytes:
            break
        header_bytes += _HEADER_BYTES
    tmp = str(path) + ".tmp"
    with open(tmp, "wb") as fh:
        fh.write(blob.ljust(header_bytes, b"\0"))
        for name, _ in _ARRAYS:
            if name not in table:
                continue
            fh.seek(table[name]["offset"])
            np.ascontiguousarray(arrs[name], dtype=table[name]["dtype"]).tofile(fh)
        fh.truncate(off)
    os.replace(tmp, path)


class ProblemFile:
    """A mapped QOCOPROB 2 file: ``.data`` (ProblemData whose arrays are views of the mapping), ``.perm`` (or
    None), ``.meta``.  ``pin()`` page-locks the mapping for fast host -> device copies; ``close()`` undoes it."""

    def __init__(self, path, validate=True):
        self.path = str(path)
        with open(self.path, "rb") as fh:
            first = fh.readline()
            if first.split() != [MAGIC.encode(), str(BINARY_VERSION).encode()]:
                raise BadSparseStructure(f"unsupported problem file header: {first[:32]!r}")
            try:
                head = json.loads(fh.readline().decode())
            except ValueError as e:
                raise BadSparseStructure(f"malformed binary problem header: {e}") from None
        self.meta = head.get("meta", {})
        self._map = np.memmap(self.path, dtype=np.uint8, mode="r")
        size = self._map.size

        def view(name):
            t = head["arrays"].get(name)
            if t is None:
                return None
            dt = np.dtype(t["dtype"])
            end = t["offset"] + t["count"] * dt.itemsize
            if t["offset"] % _ALIGN or end > size:
                raise BadSparseStructure(f"array {name} lies outside the file")
            return self._map[t["offset"]:end].view(dt)

        mats = {}
        for k in "PAG":
            r, c = head["shapes"][k]
            mats[k] = SparseMatrixCSC(int(r), int(c), view(k + "_p"), view(k + "_i"), view(k + "_x"))
        cone = ConeSpec(int(head["l"]), tuple(int(q) for q in view("soc_dims")))
        self.data = ProblemData(int(head["n"]), int(head["m"]), int(head["p"]), mats["P"], view("c"), mats["A"],
                                view("b"), mats["G"], view("h"), cone)
        self.perm = view("perm")
        self._pinned = False
        if validate:
            validate_problem(self.data)

    def pin(self, device: int = 0) -> bool:
        """Page-lock the mapping (cudaHostRegister, read-only).  Returns False when the driver refuses (e.g. the
        locked-memory limit); the file is still usable, copies are then staged by the driver."""
        from . import _lib

        lib = _lib.require_device(device)
        if not self._pinned:
            self._pinned = lib.qs_host_register(self._map.ctypes.data, self._map.size) == 0
        return self._pinned

    def close(self):
        if self._pinned:
            from . import _lib

            _lib.load().qs_host_unregister(self._map.ctypes.data)
            self._pinned = False

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ------------------------------------------------------------------ front end
def _is_binary(path) -> bool:
    with open(path, "rb") as fh:
        return fh.readline().split() == [MAGIC.encode(), str(BINARY_VERSION).encode()]


def save_problem(data: ProblemData, path, binary: bool | None = None, perm=None, meta=None) -> None:  # fileio.py:62-64
    if binary is None:
        binary = str(path).endswith(".qp2")
    if binary:
        save_problem_binary(data, path, perm=perm, meta=meta)
    else:
        with open(path, "w") as fh:
            fh.write(problem_to_text(data))


def load_problem(path) -> ProblemData:  # fileio.py:120-122
    if _is_binary(path):
        return ProblemFile(path).data
    with open(path) as fh:
        return problem_from_text(fh.read())
