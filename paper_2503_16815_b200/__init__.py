"""B200-native DeFT data-parallel hot path.

Drop-in for the scheduling / solver / preserver API of the reference package
``deftsim`` (re-export surface of deftsim/__init__.py:10-98, minus the
simulator, trace reconstruction and CLI, which are outside the hot path),
plus the executor that runs the schedule on real GPUs:

  * ``naive_knapsack`` / ``recursive_knapsack`` -> sm_100a batched bitset DP
    (csrc/subset_sum.cu) through the C-ABI in include/deft_b200.h;
  * bucket reduce + delayed SGD/momentum update -> NVLink P2P kernels
    (csrc/bucket_comm.cu), driven by ``DeftDataParallel``.
"""
from .errors import (ComparisonError, DeftError, DegenerateDistributionError, DeviceError,
                     InfeasiblePartitionError, InternalInvariantError, MalformedTraceError,
                     NonSteadyStateError, ProfileValidationError, ReconstructionError,
                     ScheduleMismatchError, SchemaError, ValidationError)
from .knapsack import (MAX_EXACT_CAPACITY, Item, KnapsackAssignment, brute_force_multi_knapsack,
                       greedy_multi_knapsack, naive_knapsack, recursive_knapsack)
from .partition import (DEFAULT_PARTITION_SIZE, PartitionConfig, comm_capacity_bound_us,
                        fuse_buckets, partition_buckets, partition_by_size)
from .experiment import RunReport, compare, emit_reports, load_experiment_config
from .preserver import (BatchSequence, ConvergenceVerdict, WalkParams, baseline_expected_state,
                        check_sequence, expected_next_state, extract_batch_sequence,
                        feedback_loop, sequence_expected_state)
from .profiles import (BucketProfile, ClusterSpec, LinkSpec, ModelProfile, cluster_from_dict,
                       cluster_to_dict, comm_time_on_link, coverage_rate, load_cluster,
                       load_profile, multi_link_coverage_rate, profile_from_dict,
                       profile_to_dict, save_profile)
from .scheduler import (SCHEMES, CapacityModel, Case, DeftScheduler, ExecNote, QueueState,
                        Schedule, ScheduleDecision, Transfer, UpdateEvent,
                        baseline_nonsequential, baseline_priority, baseline_wfbp,
                        build_schedule, deft_schedule, effective_update_frequency,
                        run_lockstep, sync_schedule_time_us)

__version__ = "0.1.0"


def __getattr__(name):
    # the executor pulls in torch; import it lazily so the solver API stays light
    if name in ("DeftDataParallel", "DeftConfig"):
        from . import executor
        return getattr(executor, name)
    if name in ("LoopbackWorld", "LoopbackRank"):
        from . import loopback
        return getattr(loopback, name)
    raise AttributeError(name)
