"""B200-native BlockBatch batched denoising step (arXiv 2605.29233).

Drop-in for the reference ``blockbatch`` generate/branch API
(``/root/reference/pkg/src/blockbatch/__init__.py:5-12``): the same names,
argument meanings and error types, with the hot path — the batched
denoising step — running as hand-written sm_100a CUDA kernels behind the
C-ABI library ``libbb200.so`` (include/bb200.h).  There is no CPU fallback:
anything that computes needs the library and a B200.
"""

from .decoding import (DecodeConfig, GenerationResult, NfeCounter, TraceEvent, BranchState,
                       confidence_transition, single_branch_decode, vanilla_decode)
from .errors import ConfigError, ContractError, RunawayError, StateError
from .model import (BlockWindow, DenoiseOutput, KvCache, ModelDims, ModelParams, SequenceRow, Task, Vocab,
                    block_forward, build_model, full_forward, kv_vectorize, make_task, exact_match, serialize_params,
                    LLADA_8B, LLADA_8B_VOCAB, DREAM_7B, DREAM_7B_VOCAB)
from .scheduler import (PackedQuery, SchedulerConfig, batched_block_forward, get_active_branches, init_full_forward,
                        merge_sync, pack_active_blocks, read_trace, run_blockbatch, run_batch, select_eos_winner,
                        write_trace, summary_row, write_summary, generated_tokens)

__version__ = "0.1.0"
