"""B200-native TIE score / rank / fit path (arXiv 2604.00499).

Drop-in for the reference's ``tiesched`` Python package on the hot path
(proj/python/tiesched/__init__.py re-exports ``_core``): the same names --
``McContext``, ``LogTParams``, ``CensoredLogT``, ``censored_expectation``, ``censored_cvar``,
``ScoreConfig``, ``compute_beta``, ``compute_score``, ``fit_logt_fixed_nu`` ... -- backed by
hand-written sm_100a kernels through the C-ABI in ``include/tie_cuda.h``, plus batched
entry points (``score_batch``, ``rank``, ``score_rank``, ``fit_logt_fixed_nu_batch``) and
device-pointer entry points for torch CUDA tensors (``paper_2604_00499_b200.torch_api``).

There is no CPU fallback: importing without the built extension raises.
"""
from __future__ import annotations

import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libtie_b200.so")
INCLUDE_DIR = os.path.join(os.path.dirname(_HERE), "include")

try:
    from ._core import *  # noqa: F401,F403
    from ._core import __version__  # noqa: F401
    from . import _core
except ImportError as exc:  # pragma: no cover - exercised only on a broken build
    raise ImportError(
        "paper_2604_00499_b200: the CUDA extension is not built "
        f"({exc}); run `python -c 'import __graft_entry__ as g; g.build()'` "
        "or `make -C paper_2604_00499_b200/csrc`"
    ) from exc


def loaded_library_path() -> str:
    """Path of the native library this process loaded (for load-evidence checks)."""
    return LIB_PATH
