"""B200-native ACDC structured linear layer (arXiv 1511.05946).

Drop-in replacement for the reference package's forward / backward /
parameter-gradient hot path: the layer API mirrors ``acdc.layers`` and runs
on hand-written sm_100a kernels behind the C ABI in ``include/acdc_b200.h``.
No CPU fallback: without ``libacdc_b200.so`` (``python -m
paper_1511_05946_b200.build``) and a CUDA device, every numeric call raises.
"""

from .functional import (
    AcdcFunction,
    AfdfFunction,
    acdc,
    acdc_backward,
    acdc_forward,
    afdf,
    afdf_backward,
    afdf_forward,
    dct,
    idct,
    prepare,
)
from .layers import (
    AcdcLayer,
    AfdfLayer,
    Cascade,
    DenseLayer,
    Layer,
    Param,
    PermutationLayer,
    ReluLayer,
    acdc_cascade,
    afdf_cascade,
    count_params,
    load_cascade,
    save_cascade,
)
from .plans import DctPlan, FftPlan, dct_matrix, resolve_backend

__version__ = "0.1.0"
