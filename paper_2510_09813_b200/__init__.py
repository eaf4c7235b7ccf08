"""B200-native state-vector hot path for the rydsim neutral-atom emulator (arxiv 2510.09813, emu-sv).

Drop-in mirror of the reference's state-vector interfaces
(rydsim.hamiltonian / rydsim.krylov / rydsim.sv / rydsim.observables / rydsim.pulses)
whose arithmetic runs in hand-written sm_100a kernels behind the C ABI in
``include/rsv.h`` (``_rsv.so``). There is no CPU fallback.
"""

__version__ = "0.1.0"

from .errors import (  # noqa: F401
    REFERENCE_ERRORS,
    ConfigurationError,
    MemoryBudgetError,
    RydsimError,
    SolverError,
    ValidationError,
)
from .hamiltonian import (  # noqa: F401
    HamiltonianSlice,
    Register,
    apply_hamiltonian,
    build_dense,
    build_diagonal,
    interaction_diagonal,
    interaction_matrix,
    weighted_bit_sum,
)
from .krylov import KrylovConfig, KrylovReport, expm_multiply  # noqa: F401
from .observables import (  # noqa: F401
    ObservableRecord,
    ObservableSpec,
    correlation,
    fidelity,
    norm_difference,
    occupation,
    occupations,
    overlap,
    sample_bitstrings,
)
from .pulses import (  # noqa: F401
    Blackman,
    ChannelProgram,
    Constant,
    DiscretizedSequence,
    InterpolatedSpline,
    Ramp,
    SampledSequence,
    discretize,
    sample_program,
    sample_waveform,
)
from .sv import SvRunConfig, SvRunResult, evolve_sv, memory_estimate_sv  # noqa: F401
