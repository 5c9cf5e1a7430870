"""CPU-only checks of the C ABI: the library loads, exports every symbol that
include/vjp.h declares, and its host-only entry points (workspace queries,
argument validation, the multi-GPU carry combination) behave — no compute call
needs a GPU here."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2202_10297_b200 import _build

    _build.build()
    import paper_2202_10297_b200 as vjp

    return vjp.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "vjp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(vjp_[a-z_0-9]+)\s*\(", src)))


def test_exports(L):
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, f"declared in include/vjp.h but not exported: {missing}"


def test_status_strings(L):
    for code in range(8):
        assert L.vjp_status_string(code).decode().startswith("VJP_")


def test_scan_workspace_query(L):
    # one tile of f64 ADD holds 256 rows x 16 elements; the workspace grows with the tile count
    a = L.vjp_scan_workspace_bytes(1, 2, 4096 * 100)
    b = L.vjp_scan_workspace_bytes(1, 2, 4096 * 1000)
    assert 0 < a < b
    assert L.vjp_scan_workspace_bytes(99, 2, 10) == 0  # bad tag
    assert L.vjp_scan_partial_bytes(6, 2) == (4 + 8) * 8  # MAT2 record: fwd 2x2 + reverse map (D, C)
    assert L.vjp_scan_partial_bytes(5, 2) == (2 + 3) * 8  # LINREC: (D, C) + (D0, D1, C)


def test_scan_argument_validation_without_gpu(L):
    buf = (ctypes.c_double * 64)()
    p = ctypes.addressof(buf)
    p16 = p + (16 - p % 16) % 16
    # n < 0
    assert L.vjp_scan(1, 2, -1, None, ctypes.c_void_p(p16), ctypes.c_void_p(p16 + 256), None, None, 0, None, 0) == 1
    # bad dtype
    assert L.vjp_scan(1, 7, 4, None, ctypes.c_void_p(p16), ctypes.c_void_p(p16 + 256), None, None, 0, None, 0) == 1
    # missing `as` for MAT2
    assert L.vjp_scan(6, 2, 4, None, ctypes.c_void_p(p16), ctypes.c_void_p(p16 + 256), None, None, 0, None, 0) == 1
    # misaligned pointer
    assert L.vjp_scan(1, 2, 4, None, ctypes.c_void_p(p16 + 8), ctypes.c_void_p(p16 + 256), None, None, 0, None,
                      0) == 7
    # workspace too small
    assert L.vjp_scan(1, 2, 4, None, ctypes.c_void_p(p16), ctypes.c_void_p(p16 + 256), None, None, 0, None, 0) == 3
    # n == 0 is a no-op
    assert L.vjp_scan(6, 2, 0, None, None, None, None, None, 0, None, 0) == 0


# --------------------------------------------------------------------------
# multi-GPU carry combination (vjp_scan_finish's device prologue, host build)
# --------------------------------------------------------------------------

def _records_mat2(A, Y, bounds):
    """per-shard record [fwd product (4) | reverse map (D 4, C 4)], computed from
    the definitions: forward = product of the shard's matrices (R1);
    reverse map X -> D + X C is the shard's composition of
    H_i = (ybar_i + H_{i+1}) A_i^T (the recurrence of P:1180, grouped per element)."""
    recs = []
    for s, e in bounds:
        P = np.eye(2)
        for i in range(s, e):
            P = P @ A[i]
        D = np.zeros((2, 2))
        C = np.eye(2)
        for i in range(e - 1, s - 1, -1):
            D = (Y[i] + D) @ A[i].T
            C = C @ A[i].T
        recs.append(np.concatenate([P.ravel(), D.ravel(), C.ravel()]))
    return np.stack(recs)


def test_carries_host_mat2_against_oracle(L):
    rng = np.random.default_rng(0)
    n, world = 40, 4
    A = rng.random((n, 2, 2)) * 0.5
    Y = rng.random((n, 2, 2))
    bounds = [(r * n // world, (r + 1) * n // world) for r in range(world)]
    recs = np.ascontiguousarray(_records_mat2(A, Y, bounds))
    _, ys = oracle.vjp_scan("mat2", Y.ravel(), A.ravel(), want_ys=True)
    ys = ys.reshape(n, 2, 2)
    for r in range(world):
        fwd = np.zeros(4)
        rev = np.zeros(4)
        rc = L.vjp_scan_carries_host(6, 2, r, world, recs.ctypes.data_as(ctypes.c_void_p),
                                     fwd.ctypes.data_as(ctypes.c_void_p), rev.ctypes.data_as(ctypes.c_void_p))
        assert rc == 0
        s, e = bounds[r]
        exp_fwd = ys[s - 1].ravel() if s > 0 else np.eye(2).ravel()
        np.testing.assert_allclose(fwd, exp_fwd, rtol=1e-13)
        # reverse carry = H entering shard r from the right = sum over later j of
        # ybar_j A_j^T ... A_{e}^T  (brute force)
        H = np.zeros((2, 2))
        for j in range(n - 1, e - 1, -1):
            H = (Y[j] + H) @ A[j].T
        np.testing.assert_allclose(rev, H.ravel(), rtol=1e-12, atol=1e-300)


def test_carries_host_add(L):
    rng = np.random.default_rng(1)
    world = 3
    sums = rng.random(world)
    recs = np.stack([np.array([0.0, s]) for s in sums])  # [fwd (unused) | D]
    for r in range(world):
        fwd, rev = np.zeros(1), np.zeros(1)
        assert L.vjp_scan_carries_host(1, 2, r, world, recs.ctypes.data_as(ctypes.c_void_p),
                                       fwd.ctypes.data_as(ctypes.c_void_p),
                                       rev.ctypes.data_as(ctypes.c_void_p)) == 0
        assert rev[0] == pytest.approx(sums[r + 1:].sum(), rel=1e-15)


def test_extension_entry_points_validate_without_gpu(L):
    """vjp_scan_batched / vjp_kmeans / vjp_scan_partial2 / the general reduce
    reject bad arguments before any launch (no GPU needed)."""
    vp = ctypes.c_void_p
    buf = (ctypes.c_double * 64)()
    p = ctypes.addressof(buf)
    p16 = vp(p + (16 - p % 16) % 16)
    # workspace queries
    assert L.vjp_scan_batched_workspace_bytes(1, 2, 1000, 8) > 0
    assert L.vjp_scan_batched_workspace_bytes(3, 2, 1000, 8) > 0       # MIN batched is offered
    assert L.vjp_scan_batched_workspace_bytes(1, 2, 1000, 0) == 0      # width < 1
    assert L.vjp_kmeans_workspace_bytes(2, 1000, 16, 8) > 0
    assert L.vjp_kmeans_workspace_bytes(2, 1000, 0, 8) == 0
    assert L.vjp_reduce_workspace_bytes(6, 2, 1000) > 0                # MAT2: the general rule's workspace
    # argument errors
    assert L.vjp_scan_batched(1, 2, 10, 0, None, p16, p16, p16, 1 << 20, None, 0) == 1   # width 0 -> EINVAL
    assert L.vjp_scan_batched(9, 2, 10, 2, None, p16, p16, p16, 1 << 20, None, 0) == 1   # bad tag
    assert L.vjp_scan_batched(5, 2, 10, 2, None, p16, vp(p16.value + 256), p16, 1 << 20, None, 0) == 1  # LINREC needs as
    assert L.vjp_kmeans(2, 10, 0, 4, p16, p16, p16, p16, None, None, None, None, p16, 1 << 20, None, 0) == 1
    assert L.vjp_kmeans(2, 10, 20_000, 4, p16, p16, p16, p16, None, None, None, None, p16, 1 << 20, None, 0) == 2
    assert L.vjp_kmeans(2, 10, 4, 4, p16, p16, p16, p16, None, None, None, None, p16, 0, None, 0) == 3  # workspace
    from paper_2202_10297_b200 import VjpShard
    sh = VjpShard(0, 2, 0, 20)
    assert L.vjp_scan_partial2(1, 2, 10, None, p16, p16, 1 << 20, sh, p16, p16, None, 0) == 2  # ADD: one exchange
    sh1 = VjpShard(0, 1, 0, 10)
    assert L.vjp_scan_partial2(3, 2, 10, p16, p16, p16, 1 << 20, sh1, p16, p16, None, 0) == 1  # world 1
    assert L.vjp_reduce(6, 2, 10, None, p16, p16, None, None, p16, 1 << 20, None, 0) == 1    # MAT2 needs as


def test_header_is_plain_c_and_links(tmp_path, L):
    """include/vjp.h is a C (not C++) header and a C program links against
    libvjp_b200.so through it (no torch types in the boundary)."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    src = tmp_path / "abi.c"
    src.write_text('#include "vjp.h"\n#include <stdio.h>\n'
                   'int main(void) { printf("%s\\n", vjp_status_string(VJP_EINVAL));\n'
                   '  return vjp_scan_workspace_bytes(VJP_ADD, VJP_F64, 0) == (size_t)-1; }\n')
    libdir = os.path.join(ROOT, "paper_2202_10297_b200", "_lib")
    exe = tmp_path / "abi"
    subprocess.check_call(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), str(src),
                           "-L", libdir, "-lvjp_b200", "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True, env={**os.environ, "LD_LIBRARY_PATH": libdir})
    assert out.returncode == 0 and out.stdout.startswith("VJP_EINVAL"), (out.returncode, out.stdout, out.stderr)
