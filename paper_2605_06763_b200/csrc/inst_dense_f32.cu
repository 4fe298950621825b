// Query-kernel instantiations: T=float, mode=kDense, DP in {64,128,256}, G in {1,2,4,8}.
#include "louver_dispatch.h"

namespace lvk {
LVK_DEFINE_LAUNCH_ALL(float, kDense)
}  // namespace lvk
