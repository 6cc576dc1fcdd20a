// capi_internal.hpp -- the opaque handle's definition, shared by the C-ABI
// translation units (capi.cpp, staged.cpp).
#pragma once
#include "llama_b200.h"
#include "mapping.hpp"

struct llama_mapping {
  llb::Mapping m;
};

namespace llb {
llama_status set_error(llama_status s, const std::string& msg);  // thread-local last error
}
