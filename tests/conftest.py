import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long CPU case (still part of the default suite unless deselected)")


# ---- the chi = 1024 oracle (several CPU minutes) runs in a background thread from the moment the
# session has collected the test that needs it, so it overlaps the rest of the GPU suite (the ctypes
# call releases the GIL). tests/test_gpu_slow_chi1024.py joins it.
_BG = {}


def background_oracle(key):
    """The (spectrum, record) the background thread computed for `key` (joins the thread)."""
    t = _BG.get(key)
    if t is None:
        return None
    t["thread"].join()
    if "error" in t:
        raise t["error"]
    return t["result"]


def _start_chi1024_oracle():
    import threading

    def work(slot):
        try:
            import numpy as np

            import oracle
            import workloads
            tensors, gates = workloads.micro_chain(1024, 1)
            o = oracle.OracleMPS(2, strategy="fixed", f_fixed=0.9999)
            o.import_site(0, tensors[0])
            o.import_site(1, tensors[1])
            o.apply_layer(np.zeros(1, np.int32), gates)
            slot["result"] = (o.last_spectrum(0), o.records()[0])
        except Exception as e:  # re-raised in the test
            slot["error"] = e

    slot = {}
    slot["thread"] = threading.Thread(target=work, args=(slot,), daemon=True)
    slot["thread"].start()
    _BG["chi1024"] = slot


def pytest_collection_finish(session):
    if any("chi1024" in it.nodeid for it in session.items):
        _start_chi1024_oracle()
