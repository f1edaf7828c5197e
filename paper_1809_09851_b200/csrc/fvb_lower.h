// fvb_lower.h -- internal: the general-lowering fallback of fvb_lookup.
#pragma once

#include "fvb.h"

namespace fvb {

// Lower a well-formed structural key to one NVRTC-compiled sm_100a kernel
// (fvb_lower.cu); cached per key.
fvb_status lower_lookup(const char* key, fvb_kernel* out);

}  // namespace fvb
