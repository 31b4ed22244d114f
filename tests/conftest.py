import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a); parity tests proper")
    config.addinivalue_line("markers", "slow: takes more than a few seconds on CPU")


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    """Report how often the C6 rank window was used."""
    try:
        import gpu_util
    except Exception:
        return
    if gpu_util.WINDOW_CHECKS[0] == 0:
        return
    tr = terminalreporter
    tr.write_line(f"rank-window: {gpu_util.WINDOW_CHECKS[0]} rank comparisons, "
                  f"{len(gpu_util.WINDOW_HITS)} split(s) accepted inside 1e-12 tau + c_floor u s(x)")
    for h in gpu_util.WINDOW_HITS:
        tr.write_line(f"  window hit {h[0]} split {h[1]}: gpu {h[2]} oracle {h[3]} |tail-tau|/window {h[4]:.3g}")
