"""paper_2103_03330_b200 -- direct GPU zero-copy feature gather for GCN minibatches (B200).

B200-native rebuild of the hot path of arXiv 2103.03330 (PyTorch-Direct): layered uniform
sampling on the GPU and the sparse feature gather that reads rows of a pinned, mapped host
table over PCIe with zero-copy loads and writes them densely into HBM.  The compute is in
``libdgz.so`` (CUDA, sm_100a; C ABI in ``include/dgz.h``); ``dgz`` is its thin binding (it
raises ImportError when libdgz.so is missing: there is no fallback) and ``pipeline`` the
per-GPU minibatch fetcher (ping-pong buffers, side stream).
"""
import importlib


def __getattr__(name):
    if name in ("dgz", "pipeline"):
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
