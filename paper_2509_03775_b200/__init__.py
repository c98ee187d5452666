"""B200-native ContraGS training hot path (drop-in for `contrags` 0.1.0's render /
train-step / MCMC-step API; reference `pkg/src/contrags/__init__.py:10-27`).

State lives in HBM as torch tensors; every compute entry point runs the
hand-written sm_100a kernels of ``libcgs_b200.so`` through its C ABI
(include/cgs_b200.h).  There is no CPU fallback.
"""

from .camera import Camera, look_at, ring_cameras
from .metrics import LossTerms, evaluate, psnr, recon_loss, recon_loss_grad, ssim, total_loss
from .modelio import (ModelFormatError, deserialize_model, image_to_u8, load_model, quantize8,
                      save_model, serialize_model, write_metrics_csv)
from .model import (Codebook, GaussianArrays, ModelState, densify, init_one_to_one, lookup,
                    model_bytes, remap_gaussian, sh_dim, validate_state)
from .render import (Frame, GradientSet, ProjectedSplat, RenderArtifacts, build_covariance,
                     project_gaussian, rasterize_backward, rasterize_forward, render_frame,
                     render_u8)
from .reassign import mutual_pairs, nearest_codes, reassign_codes
from .sampler import (MergeProposal, SamplerConfig, SamplerError, SplitProposal,
                      TransitionRecord, accept_merge, accept_split, acceptance_probability,
                      apply_merge, apply_split, choose_transition, propose_merge, propose_split,
                      q_sm, sgld_update, train, train_step)

__version__ = "0.1.0"
