import os
import sys

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity run")


def pytest_sessionfinish(session, exitstatus):
    """Dump the achieved parity errors (casebuild.PARITY_LOG) when
    DG_PARITY_LOG names a file."""
    path = os.environ.get("DG_PARITY_LOG")
    if not path:
        return
    try:
        import casebuild
    except Exception:
        return
    if not casebuild.PARITY_LOG:
        return
    import json
    import platform
    with open(path, "w") as f:
        json.dump({"host": platform.node(), "exitstatus": int(exitstatus),
                   "checks": casebuild.PARITY_LOG}, f, indent=1)
