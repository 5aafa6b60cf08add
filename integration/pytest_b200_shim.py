"""pytest plugin: install integration.gpu_weights into the reference package
before its test modules import it, and report libmlb's launch count.

    python -m pytest -p integration.pytest_b200_shim <multilap tests>
"""

_start = [0]


def pytest_configure(config):
    import multilap

    from integration import gpu_weights
    gpu_weights.install(multilap)
    _start[0] = gpu_weights.launches()


def pytest_sessionfinish(session, exitstatus):
    from integration import gpu_weights
    print(f"\n[b200-shim] libmlb kernel launches during the reference tests: {gpu_weights.launches() - _start[0]}")
