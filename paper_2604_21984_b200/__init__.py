"""B200-native SAD (Soft Anisotropic Diagrams, arXiv 2604.21984) fitting loop.

The hot path (top-K propagation, softmax blend, analytic backward with per-site reduction, Adam,
densify/prune, the resident fit) runs as hand-written sm_100a CUDA kernels in the in-tree library
`libsad_b200.so` behind the C ABI `include/sad_b200.h`.  This package mirrors the reference
library's `sad::` API on top of it; there is no CPU fallback.
"""
from .types import (AdamState, CandidateField, FitResult, GradBuffer, HistoryRow, ImageBuffer, PassSpec,  # noqa
                    RefreshMode, RunOpts, Site, SiteStats, SiteStore, StatsResult, Stencil, TrainConfig,
                    history_line, normalization_scale, psnr_from_loss, run_opts, kGradSlots, kChannels)
from .api import (Backend, CudaError, EmptyList, InvalidArgument, NumericError, StaleField,  # noqa
                  ResidentField, ResidentSites, gpu_backend, load_library, LIB_PATH)
