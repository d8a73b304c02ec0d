"""paper_2105_08764_b200 -- B200-native (sm_100a) hot path of OpenGraphGym-MG.

Drop-in for the reference `graphrl` package's parallel RL inference/training
step: the same public names and signatures, with the numerics in libs2v.so
(hand-written CUDA for sm_100a behind a C ABI, include/s2v.h) and the node
shards resident in HBM.  There is no CPU compute path.
"""
from .agent import (ExperienceTuple, MetricsRow, ReplayBuffer, TrainConfig, act, batch_targets,
                    compute_target, evaluate_ratio, load_train_state, pack_solution,
                    save_train_state, train, train_step, tuples_to_graphs, unpack_solution)
from .collective import Comm, CollectiveStats, DistComm, WorkerGroup, run_workers
from .env import MVC, PROBLEMS, MvcEnv, ProblemSpec, reset
from .errors import (CollectiveAborted, CollectiveError, ConfigError, DataError, GraphRLError,
                     InvalidActionError)
from .graphs import (Graph, generate_ba, generate_er, generate_rmat, is_vertex_cover,
                     load_edge_list, write_edge_list)
from .inference import SelectionSchedule, SolveResult, select_top_d, solve
from .policy import (PARAM_NAMES, AdamState, PolicyParams, adam_step, embed_forward,
                     load_checkpoint, loss_and_gradients, masked_scores, param_shapes, q_forward,
                     save_checkpoint, zero_grads)
from .state import Partition, PartitionedState, apply_action, is_covered, partition_rows

__version__ = "0.1.0"
