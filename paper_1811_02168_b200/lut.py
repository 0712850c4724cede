"""Lookup table of optimal (K*, T*) over a (sigma, log10(1/eps)) grid
(the reference's include/fourierbf/lut.hpp, src/lut.cpp).

build_lut runs Algorithm 1 per cell through fbf_build_lut (the period scans on
the GPU when `device` is given: identical cells, see fbf_scan.cu); query_lut
interpolates through fbf_query_lut; the text format, load/save and the trend
check are host file logic restated here.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .fbf import FBF_EUNREACHABLE, FbfError, InvalidArgument, _check, _dptr


class LutRangeError(FbfError):
    """std::out_of_range of query_lut (lut.cpp:120,125)."""


@dataclass
class LookupTable:
    """lut.hpp:14-24."""
    dynamic_range: int = 0
    sigma_grid: list = field(default_factory=list)
    logeps_grid: list = field(default_factory=list)  # log10(1/eps), ascending
    terms: list = field(default_factory=list)        # K*[sigma][logeps]
    half_period: list = field(default_factory=list)  # T*[sigma][logeps]

    def rows(self) -> int:
        return len(self.sigma_grid)

    def cols(self) -> int:
        return len(self.logeps_grid)


@dataclass
class LutQuery:
    terms: int = 0
    half_period: int = 0


@dataclass
class TrendViolation:
    axis: str
    row: int
    col: int
    detail: str


def build_lut(sigmas, epsilons, dynamic_range: int = 255, t_max: int = 0, threads: int = 1,
              device: int | None = None) -> LookupTable:
    """lut.cpp:61-113."""
    s = np.ascontiguousarray(sigmas, dtype=np.float64)
    e = np.ascontiguousarray(epsilons, dtype=np.float64)
    K = np.zeros(s.size * e.size, dtype=np.int32)
    T = np.zeros_like(K)
    ip = ctypes.POINTER(ctypes.c_int)
    rc = _lib.load().fbf_build_lut(_dptr(s), s.size, _dptr(e), e.size, dynamic_range, t_max,
                                   -1 if device is None else int(device), threads,
                                   K.ctypes.data_as(ip), T.ctypes.data_as(ip))
    if rc == FBF_EUNREACHABLE:
        raise FbfError(_lib.last_error())
    _check(rc)
    n = e.size
    return LookupTable(dynamic_range, [float(v) for v in s], [float(np.log10(1.0 / v)) for v in e],
                       [[int(K[i * n + j]) for j in range(n)] for i in range(s.size)],
                       [[int(T[i * n + j]) for j in range(n)] for i in range(s.size)])


def query_lut(table: LookupTable, sigma: float, eps: float) -> LutQuery:
    """lut.cpp:116-143 (through fbf_query_lut)."""
    sg = np.ascontiguousarray(table.sigma_grid, dtype=np.float64)
    lg = np.ascontiguousarray(table.logeps_grid, dtype=np.float64)
    K = np.ascontiguousarray(table.terms, dtype=np.int32).ravel()
    T = np.ascontiguousarray(table.half_period, dtype=np.int32).ravel()
    if K.size != sg.size * lg.size or T.size != K.size:
        raise InvalidArgument("LUT: malformed table")
    ko, to = ctypes.c_int(0), ctypes.c_int(0)
    ip = ctypes.POINTER(ctypes.c_int)
    rc = _lib.load().fbf_query_lut(_dptr(sg), sg.size, _dptr(lg), lg.size, K.ctypes.data_as(ip),
                                   T.ctypes.data_as(ip), float(sigma), float(eps), ctypes.byref(ko),
                                   ctypes.byref(to))
    if rc == _lib.FBF_ERANGE:
        raise LutRangeError(_lib.last_error())
    _check(rc)
    return LutQuery(ko.value, to.value)


def _fmt(v: float) -> str:
    """%.17g (lut.cpp:37-41)."""
    return f"{v:.17g}"


def save_lut(table: LookupTable, path: str) -> None:
    """lut.cpp:145-170."""
    lines = [f"R {table.dynamic_range}", "sigma" + "".join(" " + _fmt(v) for v in table.sigma_grid),
             "logeps" + "".join(" " + _fmt(v) for v in table.logeps_grid)]
    lines += ["K" + "".join(f" {v}" for v in row) for row in table.terms]
    lines += ["T" + "".join(f" {v}" for v in row) for row in table.half_period]
    with open(path, "w", newline="\n") as f:
        f.write("\n".join(lines) + "\n")


def _ascending(grid, name):
    if len(grid) < 2:
        raise InvalidArgument(f"LUT: {name} grid needs at least two points")
    if any(not (b > a) for a, b in zip(grid, grid[1:])):
        raise InvalidArgument(f"LUT: {name} grid must be strictly ascending")


def _int_token(tok: str, line_no: int, path: str) -> int:
    try:
        if tok.strip() != tok or not tok:
            raise ValueError
        return int(tok, 10)
    except ValueError:
        raise RuntimeError(f"LUT: non-integer entry '{tok}' at line {line_no} of {path}") from None


def load_lut(path: str) -> LookupTable:
    """lut.cpp:172-244."""
    try:
        with open(path, "rb") as f:
            lines = f.read().decode("latin-1").split("\n")
    except OSError:
        raise RuntimeError(f"LUT: cannot open {path}") from None
    if lines and lines[-1] == "":
        lines.pop()
    pos = [0]

    def nxt(expect):
        if pos[0] >= len(lines):
            raise RuntimeError(f"LUT: missing {expect} line at line {pos[0] + 1} of {path}")
        line = lines[pos[0]]
        pos[0] += 1
        return line

    def tagged(line, tag):
        toks = line.split()
        got = toks[0] if toks else ""
        if got != tag:
            raise RuntimeError(f"LUT: expected '{tag}' at line {pos[0]} of {path}, got '{got}'")
        return toks[1:]

    t = LookupTable()
    toks = tagged(nxt("R"), "R")
    if not toks:
        raise RuntimeError(f"LUT: missing R value at line 1 of {path}")
    t.dynamic_range = _int_token(toks[0], pos[0], path)
    if t.dynamic_range < 1:
        raise RuntimeError(f"LUT: R must be >= 1 in {path}")

    def floats(toks):
        out = []
        for v in toks:  # istream >> double stops at the first bad token
            try:
                out.append(float(v))
            except ValueError:
                break
        return out

    t.sigma_grid = floats(tagged(nxt("sigma"), "sigma"))
    t.logeps_grid = floats(tagged(nxt("logeps"), "logeps"))
    _ascending(t.sigma_grid, "sigma")
    _ascending(t.logeps_grid, "log10(1/eps)")
    for tag, dest in (("K", t.terms), ("T", t.half_period)):
        for _ in t.sigma_grid:
            row = [_int_token(v, pos[0] + 1, path) for v in tagged(nxt(tag), tag)]
            if len(row) != len(t.logeps_grid):
                raise RuntimeError(f"LUT: row length mismatch at line {pos[0]} of {path}")
            if any(v < 1 for v in row):
                raise RuntimeError(f"LUT: non-positive entry at line {pos[0]} of {path}")
            dest.append(row)
    return t


def check_monotone_trends(table: LookupTable) -> list[TrendViolation]:
    """lut.cpp:246-266: K* nonincreasing and T* nondecreasing with sigma."""
    out = []
    for j in range(table.cols()):
        for i in range(1, table.rows()):
            if table.terms[i][j] > table.terms[i - 1][j]:
                out.append(TrendViolation("K", i, j, f"K* increased with sigma at fixed eps "
                                                     f"({table.terms[i - 1][j]} -> {table.terms[i][j]})"))
            if table.half_period[i][j] < table.half_period[i - 1][j]:
                out.append(TrendViolation("T", i, j, f"T* decreased with sigma at fixed eps "
                                                     f"({table.half_period[i - 1][j]} -> {table.half_period[i][j]})"))
    return out
