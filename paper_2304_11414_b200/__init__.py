"""B200-native PPMoE (Pipeline MoE, arXiv 2304.11414) MoE-layer hot path.

The reference's MoE-layer API (moesim.moe / moesim.collectives) over hand-written
sm_100a CUDA kernels reached through the C-ABI library lib/libppmoe.so.
"""

from .collectives import DP, EP, PP, TP, ConfigurationError, GroupSet, ProcessGroup, TrafficLedger, World, tp_groups
from .moe import (
    DispatchPlan,
    ExpertBank,
    ExpertFfn,
    GateOutput,
    GateParams,
    LayerConfig,
    MoeLayerWeights,
    PPMoELayer,
    aux_loss,
    build_dispatch_plan,
    gate_top1,
    gate_topk,
    global_batch_equivalence,
    ppmoe_forward,
    sync_gate_gradients,
)
from .dpmoe import dpmoe_forward, dpmoe_sync_gradients
from .feed import ReplicatedFeed
from .rng import Rng

__version__ = "0.1.0"

__all__ = [
    "DP", "EP", "PP", "TP", "ConfigurationError", "GroupSet", "ProcessGroup", "TrafficLedger", "World", "tp_groups",
    "DispatchPlan", "ExpertBank", "ExpertFfn", "GateOutput", "GateParams", "LayerConfig", "MoeLayerWeights",
    "PPMoELayer", "aux_loss", "build_dispatch_plan", "gate_top1", "gate_topk", "global_batch_equivalence", "ppmoe_forward",
    "sync_gate_gradients", "Rng", "dpmoe_forward", "dpmoe_sync_gradients", "ReplicatedFeed",
]
