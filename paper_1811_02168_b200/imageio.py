"""8-bit PGM I/O and kernel tables (the reference's imageio.cpp / kernels.cpp:120-139).

read_pgm returns the raw uint8 payload (the GPU path widens bytes to float on
the device, exactly as read_pgm's static_cast<double> does on the host);
write_pgm takes uint8, or float values that it rounds half away from zero and
rejects outside [0, 255] like imageio.cpp:83-89.
"""
from __future__ import annotations

import numpy as np

from .fbf import InvalidArgument


class PgmError(RuntimeError):
    pass


def _tokens(data: bytes, path: str):
    """Header tokens (whitespace separated, '#' comments), imageio.cpp:14-35."""
    i, n = 0, len(data)
    while True:
        while i < n:
            c = data[i:i + 1]
            if c == b"#":
                while i < n and data[i:i + 1] != b"\n":
                    i += 1
            elif c.isspace():
                i += 1
            else:
                break
        j = i
        while j < n and not data[j:j + 1].isspace():
            j += 1
        if j == i:
            raise PgmError(f"PGM: truncated header in {path}")
        tok = data[i:j].decode("latin-1")
        # the single whitespace byte after the token is consumed with it
        yield tok, min(j + 1, n)
        i = j + 1


def _header_int(tok: str, path: str, what: str) -> int:
    try:
        v = int(tok)
    except ValueError:
        raise PgmError(f"PGM: bad {what} '{tok}' in {path}") from None
    if v <= 0 or str(v) != tok.lstrip("+"):
        raise PgmError(f"PGM: bad {what} '{tok}' in {path}")
    return v


def read_pgm(path: str) -> np.ndarray:
    """imageio.cpp:53-80: binary P5, maxval 255 -> uint8 (H, W)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise PgmError(f"PGM: cannot open {path}") from None
    it = _tokens(data, path)
    magic, _ = next(it)
    if magic == "P2":
        raise PgmError(f"PGM: ASCII (P2) format not supported, need binary P5: {path}")
    if magic != "P5":
        raise PgmError(f"PGM: not a P5 file (magic '{magic}'): {path}")
    w = _header_int(next(it)[0], path, "width")
    h = _header_int(next(it)[0], path, "height")
    tok, pos = next(it)
    maxval = _header_int(tok, path, "maxval")
    if maxval != 255:
        raise PgmError(f"PGM: unsupported maxval {maxval} (only 8-bit, maxval 255): {path}")
    payload = data[pos:pos + w * h]
    if len(payload) != w * h:
        raise PgmError(f"PGM: truncated pixel payload in {path}")
    return np.frombuffer(payload, dtype=np.uint8).reshape(h, w).copy()


def write_pgm(img, path: str) -> None:
    """imageio.cpp:82-101."""
    a = np.asarray(img)
    if a.ndim != 2:
        raise InvalidArgument("write_pgm: expected a 2-D image")
    if a.dtype != np.uint8:
        v = np.asarray(a, dtype=np.float64)
        r = np.where(v >= 0, np.floor(v + 0.5), -np.floor(-v + 0.5))  # std::round: ties away from zero
        if not np.all((r >= 0.0) & (r <= 255.0)):
            raise ValueError("PGM: pixel outside [0,255] after rounding; clamp before writing")
        a = r.astype(np.uint8)
    h, w = a.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{w} {h}\n255\n".encode())
        f.write(np.ascontiguousarray(a).tobytes())


def read_kernel_table(path: str) -> np.ndarray:
    """kernels.cpp:120-139: one value per non-empty line."""
    vals = []
    try:
        lines = open(path).read().split("\n")
    except OSError:
        raise RuntimeError(f"kernel table: cannot open {path}") from None
    for no, line in enumerate(lines, 1):
        if not line:
            continue
        try:
            vals.append(float(line.split()[0]))
        except (ValueError, IndexError):
            raise RuntimeError(f"kernel table: bad value at line {no} of {path}") from None
    return np.array(vals, dtype=np.float64)
