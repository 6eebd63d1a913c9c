"""B200-native SG-PCG / NN2 solver (sm_100a CUDA behind the C ABI include/sgw.h).

The Python layer mirrors the reference sgwave solver interface for the hot
path (SgSolver / SchurSystem / pcg, include/sgwave/sg.hpp, dd.hpp, pcg.hpp)
over ctypes.  There is no CPU fallback: importing the solver requires the
compiled libsgw_b200.so and every compute call runs on the GPU.
"""
from .sgwave import (  # noqa: F401
    PRECONDS,
    DetSolver,
    ForceSpec,
    LocalGroup,
    NewmarkParams,
    SgError,
    SgInvalidArgument,
    SgHistory,
    SgOptions,
    SgSolver,
    SolveOptions,
    TimeHistory,
    TripleTensor,
    gaussian_pulse,
    lib_path,
    load_library,
    lognormal_coeff,
    nccl_unique_id,
    nearest_node,
    moments,
    precond_from_string,
    run_precond_comparison,
    ricker,
    shard_plan,
    ShardPlan,
    LocalSchur,
    SchurFromLocals,
    pcg,
    SGW_ENOCONV,
    triple_products,
    write_sg_outputs,
    kle_spectrum,
    kle_spectrum_csv,
    pce_indices,
    pce_indices_csv,
    svg_lines,
)
