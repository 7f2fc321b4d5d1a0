import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


def pytest_sessionstart(session):
    # a fresh checkout has no built libraries (they are git-ignored): build them
    # once, in-tree, when nvcc is available; an existing build is left untouched
    import shutil
    lib = os.path.join(ROOT, "paper_2312_02515_b200", "libmlora.so")
    if not os.path.exists(lib) and shutil.which("nvcc"):
        from paper_2312_02515_b200 import _build
        _build.build_all()
