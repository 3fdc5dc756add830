"""MOSEL-style modality-aware inference serving, B200-native hot path.

Drop-in for the reference ``modserve`` public API (``modserve/__init__.py:
9-31``): every name it exports is importable from here with the same
meaning.  The hot path underneath — per-job modality-subset selection,
request compaction into modality-grouped sub-batches, per-modality
encoders on tcgen05 tensor cores, late fusion + classifier head, and the
CUDA-event profiler — runs as hand-written sm_100a CUDA behind the C-ABI
library ``libmosel_b200.so`` (``include/mosel_b200.h``), loaded by
``paper_2310_18481_b200.device``.  There is no CPU fallback for it.
"""

from .planner import (Candidate, MatrixCell, MatrixError, SolverError, Strategy,
                      StrategyMatrix, all_modalities_strategy, brute_force_offline,
                      build_matrix, candidates_for_job, default_alpha_grid,
                      distinct_effective_accuracies, effective_accuracy, load_matrix,
                      recommended_alphas, save_matrix, solve_offline, strategy_latency_ms,
                      strategy_latency_us, validate_matrix)
from .policy import (FeedbackState, Job, JobQueue, JobState, Policy, ScheduleEstimate,
                     apply_policy, build_schedule_estimate, candidates_with_rounding,
                     compute_budget, detect_violation, dispatch_time_us, next_dispatch,
                     reassign_aggressive, reassign_optimized, reassign_random,
                     select_on_device, try_upgrade, update_latency_feedback)
from .records import (JobRecord, MetricsLog, Summary, WindowStats, accuracy_histogram,
                      export, read_log, summarize, window_stats)
from .registry import (ModalityCombo, ModelProfile, ProfileError, SynthSpec,
                       count_strategies, demo_profile, enumerate_combos, load_profile,
                       save_profile, scale_latency, synth_profile)
from .serving import (JobTemplate, SimConfig, SimError, TableExecutor, WorkloadError,
                      WorkloadSpec, all_modalities_capacity_qps, generate_jobs,
                      load_scenario, load_trace, map_trace_to_qps, matrix_for_jobs, run,
                      run_replicas)

__version__ = "0.1.0"
