"""pytest plugin: run the reference's own test suite with its kernel swapped for the B200 engine.

    PYTHONPATH=baseline/_ref:integration:baseline/_ref/mrsim_tests MRSIM_B200_PRECISION=64 \
        python -m pytest baseline/_ref/mrsim_tests -p mrsim_b200_pytest

``mrsim.engine.compute_block`` (engine.py:259-310) becomes a thin client of ONE GPU process: the
plugin spawns it at start-up (a fresh interpreter, the only process that touches CUDA), and the
client sends each ``(tables, block)`` there, where ``mrsim_b200.compute_block_b200`` — the ctypes
stub over the C-ABI — runs it and returns ``(echoes, snapshots)`` or the reference's exception.
Because no test process initialises CUDA itself, the reference's process pool keeps its default
``fork`` start method (engine.py:540-595): forked workers inherit whatever ``compute_block`` the
parent holds — the GPU client, or a test's own monkeypatch (the fault-injection test,
test_engine.py:214-222) — and open their own connection to the GPU process.  The plugin is
installed before the test modules import, so ``from mrsim.engine import compute_block`` in the
tests binds the GPU client too.  At the end the GPU process's call count goes to
$MRSIM_B200_CALLS_FILE.
"""

import multiprocessing as mp
import os
import tempfile
import threading
from multiprocessing.connection import Client, Listener


def _handle(conn, lock, counter):
    import mrsim_b200

    while True:
        try:
            msg = conn.recv()
        except (EOFError, OSError):
            return
        if msg == "calls":
            conn.send(counter[0])
            continue
        tables, block = msg
        try:
            with lock:
                out = mrsim_b200.compute_block_b200(tables, block)
                counter[0] += 1
            conn.send(("ok", out))
        except Exception as exc:  # re-raised as the same reference exception type by the client
            conn.send(("err", type(exc).__name__, str(exc)))


def _serve(addr, key, ready):
    lock, counter = threading.Lock(), [0]
    with Listener(addr, authkey=key) as ls:
        ready.set()
        while True:
            conn = ls.accept()
            threading.Thread(target=_handle, args=(conn, lock, counter), daemon=True).start()


_server = {"addr": None, "key": None, "proc": None}
_client = {"pid": None, "conn": None}


def _conn():
    if _client["pid"] != os.getpid():  # a forked worker opens its own connection
        _client["conn"] = Client(_server["addr"], authkey=_server["key"])
        _client["pid"] = os.getpid()
    return _client["conn"]


def compute_block_gpu(tables, block):
    """mrsim.engine.compute_block, evaluated by the GPU process."""
    c = _conn()
    c.send((tables, block))
    reply = c.recv()
    if reply[0] == "ok":
        return reply[1]
    from mrsim.errors import InvalidParameter, MrSimError, WorkerPanic

    _, name, msg = reply
    if name == "InvalidParameter":
        raise InvalidParameter(msg)
    if name == "WorkerPanic":
        raise WorkerPanic(block.index, msg)
    raise MrSimError(f"{name}: {msg}")


def _start():
    _server["addr"] = os.path.join(tempfile.mkdtemp(prefix="mrsim_b200_"), "gpu.sock")
    _server["key"] = os.urandom(16)
    ctx = mp.get_context("spawn")
    ready = ctx.Event()
    p = ctx.Process(target=_serve, args=(_server["addr"], _server["key"], ready), daemon=True)
    p.start()
    if not ready.wait(120):
        raise RuntimeError("the GPU process did not start")
    _server["proc"] = p
    import mrsim.engine

    mrsim.engine.compute_block = compute_block_gpu


if mp.current_process().name == "MainProcess" and os.environ.get("MRSIM_B200_SERVER_CHILD") is None:
    os.environ["MRSIM_B200_SERVER_CHILD"] = "1"  # the spawned GPU process imports this module too
    _start()


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("MRSIM_B200_CALLS_FILE")
    if path and _server["addr"]:
        c = _conn()
        c.send("calls")
        with open(path, "w") as fh:
            fh.write(str(c.recv()))
