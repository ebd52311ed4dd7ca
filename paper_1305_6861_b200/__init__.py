"""paper_1305_6861_b200 — B200-native (sm_100a) Bloch event-stream engine.

A drop-in for the hot path of the spin-based MR simulator of arXiv 1305.6861
(ParSpin; reference package ``mrsim``): per-isochromat integration of the Bloch
equation through the event stream plus the receive-weighted ADC sum, behind the
reference's own ``compute_block`` / ``run`` API.  The arithmetic runs in
``libbloch_b200.so`` (hand-written CUDA for sm_100a, C-ABI in
``include/bloch_b200.h``); this package is the host layer.
"""

from .bloch import GAMMA_PROTON, FrameContext, HardPulse, Magnetization, RelaxationParams, equilibrium, hard_pulse_matrix
from .engine import (
    BlochEngine,
    EchoRecord,
    EsTable,
    Experiment,
    OperatorTables,
    RunMetrics,
    RunResult,
    SpinBlock,
    build_spin_arrays,
    compare_results,
    compute_block,
    delta_e_stoer,
    flatten_tables,
    get_engine,
    partition_blocks,
    precompute_sequence_tables,
    run,
    simulate_spin,
)
from .errors import (
    DeviceError,
    FitDiverged,
    InvalidParameter,
    MrSimError,
    ParseError,
    SpinBudgetExceeded,
    TimingInfeasible,
    TrajectoryMismatch,
    WorkerPanic,
)
from .recon import ImageVolume, KSpaceMatrix, assemble_kspace, cpmg_fit, reconstruct
from .phantom import Phantom, PhantomBox, SpinSample, rasterize, rasterize_arrays, shepp_logan, shepp_logan_m0
from .sequence import (
    AcquisitionSpec,
    ElementarySequence,
    GradientWaveform,
    Sequence,
    build_cpmg,
    build_gradient_epi,
    build_spin_echo,
    build_tse,
    expand_shaped_pulse,
    readout_duration,
    readout_gradient,
)
from .system import (
    CoilArray,
    GaussianCoil,
    StaticField,
    SystemModel,
    UniformSensitivity,
    complex_weight,
    default_system,
    spin_off_resonance,
)

__version__ = "0.1.0"
