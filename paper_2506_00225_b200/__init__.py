"""B200-native candidate-view render + scoring for ActiveSGM (arxiv 2506.00225).

The compute path is libsgm_b200.so (hand-written sm_100a CUDA behind the C ABI in
include/sgm.h); this package is the host-side mirror of the reference API.
"""
from .splatmap import (  # noqa: F401
    K_MAX_FOOTPRINT,
    PROJECTION_DTYPE,
    CameraModel,
    Frame,
    LossReport,
    LossWeights,
    ParamGradients,
    CandidatePool,
    CandidatePose,
    CandidateState,
    Context,
    GaussianMap,
    Pose,
    RenderChannels,
    RenderOptions,
    RenderOutput,
    SemanticGaussian,
    backward,
    bins_of_last_render,
    clipped_entropy,
    combine_scores,
    combine_scores_fisher,
    deg_to_rad,
    fisher_prior,
    fisher_set_prior,
    look_at,
    prune_pool,
    refresh_candidate_scores,
    refresh_candidate_scores_fisher,
    render,
    render_entropy,
    render_reference,
    score_candidates,
    score_candidates_fisher,
    score_poses,
    score_poses_fisher,
    sigmoid,
)
from .explore import (  # noqa: F401,E402
    Aabb,
    ExplorationMap,
    SamplingSchedule,
    VoxelState,
    fibonacci_directions,
    sample_candidates,
)
from .mapper import (  # noqa: F401,E402
    AdamParams,
    AdamState,
    DeviceFrame,
    MapperConfig,
    MapTrainer,
    optimize_map,
)
from .evaluate import (  # noqa: F401,E402
    Evaluator,
    MetricReport,
    PerClassMetric,
    evaluate,
    photometric_metrics,
    semantic_metrics,
)
