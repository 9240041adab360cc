"""``import fastsep`` for code written against the reference package.

``install_fastsep_alias()`` registers this package under the reference's
module names (``pkg/src/fastsep/__init__.py:25-43`` and the submodules its
tests import), so a caller -- or a reference-style test -- switches backends
without editing its imports:

    from paper_1903_03237_b200.compat import install_fastsep_alias
    install_fastsep_alias()
    from fastsep import SeparatorConfig, run
    from fastsep._kernels import ip_weights

Only the hot-path surface exists behind the alias (fast-mnmf, fast-mnmf-dp,
mnmf; the operator seam ``_kernels``; ``spatial``; ``stft``; ``errors``).
"""

import sys


def install_fastsep_alias(force=False):
    """Map ``fastsep`` (+ ``.separate``, ``._kernels``, ``.spatial``,
    ``.errors``, ``.stft``) to this package. Refuses to shadow an already
    imported reference ``fastsep`` unless ``force``."""
    import paper_1903_03237_b200 as pkg
    from . import errors, kernels, separate, spatial, stft

    cur = sys.modules.get("fastsep")
    if cur is not None and cur is not pkg and not force:
        raise RuntimeError("a different 'fastsep' module is already imported")
    sys.modules["fastsep"] = pkg
    for name, mod in (("separate", separate), ("_kernels", kernels), ("spatial", spatial),
                      ("errors", errors), ("stft", stft)):
        sys.modules[f"fastsep.{name}"] = mod
    return pkg


def uninstall_fastsep_alias():
    import paper_1903_03237_b200 as pkg

    if sys.modules.get("fastsep") is pkg:
        for k in [k for k in sys.modules if k == "fastsep" or k.startswith("fastsep.")]:
            del sys.modules[k]
