// The FFE program as polarisation-split pairs at N = 2048
// (dbp_block_kernel<11, kProgFFE, kTwDit, 1>, launch.h launch_polsplit) in a
// unit of its own: build.py compiles it with ptxas --register-usage-level=8,
// which schedules this kernel 1.9% faster (105.9 -> 107.9 GS/s at 2048/700),
// while the N = 4096 pairs (-0.4%) and every split-step kernel are fastest at
// the default level (profiles/r2/ab_regusage.txt, ab_ffe_unit.txt).
#include "launch.h"

namespace dbp {

cudaError_t launch_polsplit_ffe_2048(const KernelParams& kp, cudaStream_t stream) {
  return launch_polsplit<11>(kp, stream);
}

}  // namespace dbp
