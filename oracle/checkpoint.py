"""FP32 checkpoint format, written out plainly (oracle side of NEXT-3).

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py): used by tests/ to check the
CUDA path's pf_save / pf_load; shares no code with it.

PAPER.md:239-245 (§Input/Output): "the complete simulation state has to be
stored on disk, containing four phi values and two mu values per cell ...
checkpoints use only single precision".  The byte layout is SPEC.md:462-466
(type Checkpoint):

    magic "PFCP0001"; u64 NX, NY, NZ; u32 N, u32 K-1; f64 dx, f64 t;
    u64 step, u64 window_origin_z; then component-major binary32 (all phi_1,
    ..., phi_N, mu_1, mu_2), x fastest; all little endian.

Pinned in tests/test_oracle_pins.py against a hand-assembled byte fixture
(tests/golden/checkpoint_2x1x1.hex), the file-size formula of SPEC.md:481 and
the cast-identity round trip of SPEC.md:476/479.
"""
from __future__ import annotations

import struct

import numpy as np

MAGIC = b"PFCP0001"
HEADER = struct.Struct("<8sQQQIIddQQ")   # 72 bytes


class CheckpointError(Exception):
    pass


def encode(phi, mu, dx, t, step, z_origin) -> bytes:
    """phi[N, NZ, NY, NX], mu[K-1, NZ, NY, NX] (float64) -> checkpoint bytes.
    binary32 values are numpy's IEEE round-to-nearest-even casts."""
    phi = np.asarray(phi, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    n_ph, nz, ny, nx = phi.shape
    assert mu.shape[1:] == (nz, ny, nx)
    head = HEADER.pack(MAGIC, nx, ny, nz, n_ph, mu.shape[0], float(dx), float(t), int(step), int(z_origin))
    body = b"".join(np.ascontiguousarray(f, dtype="<f4").tobytes() for f in list(phi) + list(mu))
    return head + body


def decode(data: bytes):
    """checkpoint bytes -> (header dict, phi float32[N,NZ,NY,NX], mu float32[K-1,...])."""
    if len(data) < HEADER.size:
        raise CheckpointError("truncated header")
    magic, nx, ny, nz, n_ph, n_mu, dx, t, step, zo = HEADER.unpack_from(data, 0)
    if magic != MAGIC:
        raise CheckpointError("bad magic")
    n = nx * ny * nz
    need = HEADER.size + (n_ph + n_mu) * n * 4
    if len(data) < need:
        raise CheckpointError(f"truncated body ({len(data)} of {need} bytes)")
    vals = np.frombuffer(data, dtype="<f4", count=(n_ph + n_mu) * n, offset=HEADER.size)
    vals = vals.reshape(n_ph + n_mu, nz, ny, nx)
    hdr = dict(nx=nx, ny=ny, nz=nz, n_phases=n_ph, n_mu=n_mu, dx=dx, t=t, step=step, z_origin=zo)
    return hdr, vals[:n_ph].copy(), vals[n_ph:].copy()


def write_checkpoint(path, phi, mu, dx, t, step, z_origin):
    with open(path, "wb") as f:
        f.write(encode(phi, mu, dx, t, step, z_origin))


def read_checkpoint(path):
    with open(path, "rb") as f:
        return decode(f.read())
