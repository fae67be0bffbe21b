"""B200-native CAVI engine for arxiv 2401.10068 (drop-in for `tissuemix.vb`).

    from paper_2401_10068_b200 import vb, model
    state, trace = vb.vb_fit(dataset, model.default_hyperparams(4))

See DESIGN.md for the kernel design and INTEGRATION.md for the reference-side
binding.
"""

from . import linalg, model, vb  # noqa: F401
from ._lib import EXPORTS  # noqa: F401

__version__ = "0.1.0"
