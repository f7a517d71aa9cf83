import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: takes more than a few seconds on CPU")


def _cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


# Scene trees: the product builds them on the GPU (treebuild.py).  A CPU-only
# run has no device, so the seeded test scenes take their trees from the CPU
# oracle's builder instead (bit-identical trees, tests/test_gpu_treebuild.py).
if not _cuda_available():
    from oracle import tree_oracle
    from paper_2309_15417_b200 import scenes

    scenes.TREE_BUILDER = tree_oracle.build_many
