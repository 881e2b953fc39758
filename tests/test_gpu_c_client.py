"""The C ABI from C (-m gpu): tests/c/abi_client.c, compiled here with gcc (C99) against
include/mpxa.h and linked with libmpxa.so, runs alltoall (pairwise, Bruck), allgather and a persistent alltoallv
on buffers it allocates with the CUDA runtime; every received buffer must equal the oracle's
definition (bit-exact).  No Python or torch sits between the client and the library."""
import os
import subprocess

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2309_07337_b200")


def _build(tmp_path):
    exe = tmp_path / "abi_client"
    cuda = "/usr/local/cuda"
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-I" + os.path.join(ROOT, "include"), "-I" + cuda + "/include",
                           os.path.join(ROOT, "tests", "c", "abi_client.c"), "-o", str(exe),
                           "-L" + cuda + "/lib64", "-lcudart", "-L" + LIBDIR, "-lmpxa",
                           "-Wl,-rpath=" + LIBDIR, "-Wl,-rpath=" + cuda + "/lib64"])
    return exe


@pytest.mark.parametrize("p,b", [(4, 32), (8, 1000), (5, 4096 + 3)])
def test_c_client_matches_oracle(tmp_path, p, b):
    if not os.path.exists(os.path.join(LIBDIR, "libmpxa.so")):
        pytest.skip("libmpxa.so not built")
    exe = _build(tmp_path)
    a2a = synth.alltoall_sendbuf(p + b, p, b)
    ag = synth.allgather_sendbuf(p + b, p, b)
    counts = synth.cfg4_counts(p, p, 256)
    inp = tmp_path / "in.bin"
    with open(inp, "wb") as f:
        f.write(np.array([p, b], np.int64).tobytes())
        f.write(a2a.tobytes())
        f.write(ag.tobytes())
        f.write(counts.astype(np.int64).tobytes())
    out = tmp_path / "out.bin"
    res = subprocess.run([str(exe), str(inp), str(out)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    raw = out.read_bytes()
    n = p * p * b
    want_a2a = oracle.alltoall_definition(a2a)
    assert np.array_equal(np.frombuffer(raw[:n], np.uint8).reshape(p, p * b), want_a2a), "pairwise"
    assert np.array_equal(np.frombuffer(raw[n:2 * n], np.uint8).reshape(p, p * b), want_a2a), "bruck"
    assert np.array_equal(np.frombuffer(raw[2 * n:3 * n], np.uint8).reshape(p, p * b),
                          oracle.allgather_definition(ag)), "allgather"
    vsb, vrb = np.frombuffer(raw[3 * n:3 * n + 16], np.int64)
    o = 3 * n + 16
    vs = np.frombuffer(raw[o:o + p * vsb], np.uint8).reshape(p, vsb)
    vr = np.frombuffer(raw[o + p * vsb:o + p * vsb + p * vrb], np.uint8).reshape(p, vrb)
    sc = counts.astype(np.int64)
    rc = sc.T.copy()
    sd = np.zeros_like(sc); sd[:, 1:] = np.cumsum(sc, 1)[:, :-1]
    rd = np.zeros_like(rc); rd[:, 1:] = np.cumsum(rc, 1)[:, :-1]
    want_v = oracle.alltoallv_definition(vs, sc, sd, rc, rd, 8, np.full((p, vrb), 0xA5, np.uint8))
    assert np.array_equal(vr, want_v), "alltoallv"
    assert "launches" in res.stdout
