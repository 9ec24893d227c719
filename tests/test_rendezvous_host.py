"""CPU test of the peer transports' host rendezvous (comm.cpp): the
shared-memory rendezvous of DD_COMM_IPC across forked processes and the
in-process one of DD_COMM_LOCAL across threads -- every rank receives every
rank's blob in rank order for 200 back-to-back rounds, and with one rank
missing every present rank fails after DD_PEER_TIMEOUT_S instead of hanging
(the status-agreement and failure path of dd_setup / dd_destroy)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "rdv_selftest.cpp")
CSRC = os.path.join(ROOT, "paper_2508_04917_b200", "csrc")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    from paper_2508_04917_b200 import build as b
    so = b.build()
    nd = b.nccl_dir()
    out = str(tmp_path_factory.mktemp("rdv") / "rdv_selftest")
    cmd = ["g++", "-O1", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           "-I", os.path.join(nd, "include"), "-I", "/usr/local/cuda/include", SRC, "-o", out,
           so, "-Wl,-rpath," + os.path.dirname(so), "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
           "-Wl,-rpath," + os.path.join(nd, "lib"), "-L", "/usr/local/cuda/lib64", "-lcudart_static",
           "-ldl", "-lpthread", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return out


@pytest.mark.parametrize("mode,world", [("shm", 2), ("shm", 5), ("local", 3), ("local", 8)])
def test_rendezvous_rounds(exe, mode, world):
    r = subprocess.run([exe, mode, str(world)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("mode", ["shm_missing", "local_missing"])
def test_rendezvous_missing_rank_times_out(exe, mode):
    env = dict(os.environ, DD_PEER_TIMEOUT_S="1.5")
    r = subprocess.run([exe, mode, "3"], capture_output=True, text=True, timeout=60, env=env)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
