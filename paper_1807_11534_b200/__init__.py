"""B200-native restricted-domain dual TV segmentation (arXiv 1807.11534).

The product is the C-ABI CUDA library ``librds.so`` (include/rds.h, sources in ``csrc/``);
``paper_1807_11534_b200.rds`` is its thin ctypes binding and ``workloads`` the seeded input
recipe.  The binding is imported lazily so that the input recipe can be used without the
library; importing ``rds`` without a built library raises (there is no CPU fallback).
"""
__all__ = ["rds", "workloads", "build"]


def build(force: bool = False) -> str:
    from . import _build

    return _build.build(force=force)


def __getattr__(name):
    if name in ("rds", "workloads"):
        import importlib

        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
