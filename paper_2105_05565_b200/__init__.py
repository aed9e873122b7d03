"""B200-native momentum sketch-and-project ridge solver (RidgeSketch, arXiv 2105.05565).

The hot path is libridgesketch.so (CUDA, sm_100a) behind the C ABI in include/ridgesketch.h;
`ridgesketch` is its thin Python binding.  Import of the binding fails loudly when the library
is not built -- there is no CPU fallback.
"""

__all__ = ["ridgesketch", "build"]


def build(force=False):
    from . import _build
    return _build.build(force=force)
