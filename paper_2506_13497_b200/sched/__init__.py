"""Host scheduling layer mirroring the reference ``ditsim`` API (arxiv 2506.13497):
buddy GPU allocator, greedy step-granularity DoP policy, static-DoP baseline, step-granular
serving loop, workload streams and trace metrics. Decisions are bit-exact with the
reference; the serving loop additionally accepts a B200 step executor."""

from .allocator import (AllocationError, AllocationHandle, Block, ClusterTopology, GpuPool,
                        bandwidth_aware_partition, handle_from_gpu_ids)
from .engine import (EventKind, OverheadModel, RequestRecord, RequestState, RequestStatus,
                     SimResult, Simulation, SimulationError, StepExecutor, TraceRecord)
from .metrics import MetricsReport, compute_metrics, nearest_rank_percentile, normalize
from .policies import (GreedyPolicy, PromoteEntry, SchedulingPolicy, StaticDopPolicy,
                       promotion_order, update_starvation)
from .profiles import (DopTable, ProfileError, ProfileLookupError, ProfileTable, ResolutionClass,
                       change_rate, default_profile, derive_dop_table, dump_profiles,
                       estimate_execution_time,
                       load_profiles, optimal_dop)
from .workload import (ArrivalRecord, WorkloadError, WorkloadSpec, empirical_proportions,
                       generate, load_workload, save_workload, stratified_counts)
