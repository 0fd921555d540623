import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
# the parity tests compare the tensor-core engine with the SIMT fp32 reference engine as well
os.environ.setdefault("EMBER_TEST_ENGINES", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running CPU test")
