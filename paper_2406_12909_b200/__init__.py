"""B200-native (sm_100a) data-parallel MTL training hot path of a HydraGNN-style
graph foundation model, drop-in for gfmkit's model/train/comm API.

Modules mirror the reference: ``model`` (ModelConfig, ModelParams,
make_batch, forward_batch, mtl_loss, loss_and_grad, ...), ``train``
(TrainConfig, apply_update, train, DataParallelTrainer, save_checkpoint /
load_checkpoint in the GFMP format), ``ensemble`` (ensemble_predict),
``comm`` (Comm,
LocalComm, TorchComm over NCCL), ``preprocess`` (GPU radius graph,
generate_synthetic), ``schedule`` (epoch_schedule), ``records``, ``errors``.
All arithmetic runs in ``_lib/libgfm_b200.so`` (include/gfm_b200.h).
"""

__version__ = "0.1.0"
