import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def pytest_sessionfinish(session, exitstatus):
    """Write every recorded parity check (measured disagreement beside its tolerance)."""
    import json
    try:
        from tests._util import SLACK
    except Exception:
        return
    if not SLACK:
        return
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "parity_slack.json"), "w") as f:
        json.dump(SLACK, f, indent=1)


def pytest_terminal_summary(terminalreporter, exitstatus, config):
    try:
        from tests._util import SLACK
    except Exception:
        return
    if not SLACK:
        return
    worst = sorted(SLACK, key=lambda e: -e["ratio"])[:15]
    terminalreporter.write_line(f"parity slack: {len(SLACK)} checks; largest measured/tolerance ratios:")
    for e in worst:
        terminalreporter.write_line(f"  {e['ratio']:.3g}  measured {e['measured']:.3g} tol {e['tol']:.3g}  "
                                    f"{e['test']} {e['what']}")
