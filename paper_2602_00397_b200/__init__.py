"""B200-native FastForward prefill-FFN hot path (arXiv 2602.00397).

Drop-in for the reference package's hot-path API (``sparseprefill``): the
predictor, the sparse FFN, the compensator and the layer-wise scheduler keep
their names and semantics; the arithmetic runs in hand-written sm_100a
kernels (``libffwd_b200.so``) behind a C-ABI (``include/ffwd_b200.h``).
"""

from .errors import NumericError, UnsupportedError, ValidationError
from .model import LayerWeights, ModelConfig
from .predictor import (DevicePredictor, PredictorParams, default_reduced_dim, init_predictor,
                        predictor_forward, predictor_logits, predictor_scores)
from .compensator import (CompensatorParams, apply_compensation, compensator_forward,
                          default_comp_dim, init_compensator)
from .sparse import (ExpertMask, FirstBlockStatic, SubWeights, budget_to_k, build_mask,
                     hidden_column_scores, mask_from_hidden, oracle_experts, select_subweights,
                     sparse_ffn_forward, topk_indices)
from .scheduler import (AttentionMassProfile, SparsityPlan, allocate_budgets, budgets_to_topk,
                        dense_plan, load_plan, plan_from_profile, save_plan, uniform_plan)
from .costmodel import FlopsReport, ffn_path_flops, predict_prefill_flops
from .layer import (PackedLayer, dense_ffn, ffn_layer_mode, invalidate_packed, mask_indices,
                    mask_words, oracle_scores, pack_layer, predict_mask,
                    run_sparse_ffn, seq_shard, set_raster, shard_comp_cols, shard_neurons,
                    sparse_ffn_layer)

__all__ = [name for name in dir() if not name.startswith("_")]
__version__ = "0.1.0"
