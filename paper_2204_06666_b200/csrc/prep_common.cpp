#include "ehyb_common.h"

namespace ehyb {
std::string& error_slot() {
  static thread_local std::string slot;
  return slot;
}
}  // namespace ehyb

extern "C" {
EHYB_API const char* ehyb_last_error(void) { return ehyb::error_slot().c_str(); }
EHYB_API int ehyb_abi_version(void) { return 2; }
}
