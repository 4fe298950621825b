// Query-kernel instantiations: T=__nv_bfloat16, mode=kDense, DP in {64,128,256}, G in {1,2,4,8}.
#include "louver_dispatch.h"

namespace lvk {
LVK_DEFINE_LAUNCH_ALL(__nv_bfloat16, kDense)
}  // namespace lvk
