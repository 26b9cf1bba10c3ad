"""B200-native blocked separable Helmholtz solver (arXiv 1909.01299).

The product is the C-ABI library ``_lib/liblfds.so`` (include/lfds.h); ``lfds`` is its
thin Python binding.  Importing fails loudly if the library has not been built.
"""
from .lfds import MLPlan, MWPlan, MW2Plan, Plan, setup_grid, LfdsError, version  # noqa: F401
