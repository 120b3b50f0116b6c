"""paper_2306_06446_b200 — B200-native ShiftAddViT inference (arXiv 2306.06446).

Drop-in for the inference path of the reference package `shiftadd`
(/root/reference/pkg/src/shiftadd): the modules `tensor`, `quantize`,
`attention`, `moe` and `model` keep the reference's names and signatures,
while every forward runs in libshiftadd_b200.so — hand-written sm_100a CUDA
behind the C-ABI in include/shiftadd_b200.h. There is no CPU fallback.
"""

__version__ = "0.1.0"

from . import specs  # noqa: F401  (pure-python, importable without a GPU)


def __getattr__(name):
    # lazy submodule import so `import paper_2306_06446_b200` never touches CUDA
    import importlib
    if name in ("tensor", "quantize", "attention", "moe", "model", "build", "runtime", "_lib"):
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
