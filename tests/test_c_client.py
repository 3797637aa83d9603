"""include/dolb.h from plain C: a C client (tests/c/dolb_c_client.c) compiled
with gcc and linked against _lib/libdolb.so -- the way the reference's CLI and
capi tests link libdolb.so -- runs the configuration / model queries on the
CPU and, with a GPU, a tiny dolb_run."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIBDIR = os.path.join(ROOT, "paper_2506_09242_b200", "_lib")


@pytest.fixture(scope="module")
def client(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("c") / "dolb_c_client")
    subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", os.path.join(HERE, "c", "dolb_c_client.c"),
                    "-I", os.path.join(ROOT, "include"), "-L", LIBDIR, "-ldolb", f"-Wl,-rpath,{LIBDIR}",
                    "-o", exe], check=True)
    return exe


def test_c_client_queries(client):
    r = subprocess.run([client, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "BounceBack\nCOLL_TRT\nMovingBounceBack\n" in r.stdout
    assert "bytes_per_cell 164" in r.stdout
    assert 'unknown case "vortex-street"' in r.stdout


@pytest.mark.gpu
def test_c_client_run(client, tmp_path):
    r = subprocess.run([client, "gpu", str(tmp_path / "out")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "run steps 40" in r.stdout
    assert (tmp_path / "out" / "series.csv").exists()
