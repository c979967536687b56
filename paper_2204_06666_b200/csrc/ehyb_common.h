// Internal helpers shared by the host (prep.cpp) and device (*.cu) sources:
// thread-local error text behind ehyb_last_error() and the try/catch wrapper
// that turns C++ exceptions into C-ABI status codes.
#pragma once

#include "../../include/ehyb_b200.h"

#include <new>
#include <stdexcept>
#include <string>

namespace ehyb {

std::string& error_slot();  // defined in prep_common.cpp

inline int fail(const std::string& msg, int code = EHYB_EINVAL) {
  error_slot() = msg;
  return code;
}
inline int fail_oom() { return fail("out of host memory", EHYB_ENOMEM); }

#ifdef __CUDACC__
// prep_gpu.cu: pageable -> device copy through the pinned staging buffers
cudaError_t staged_h2d(void* dev, const void* host, size_t bytes);
#endif

}  // namespace ehyb

#define EHYB_TRY try
#define EHYB_CATCH                                                        \
  catch (const std::bad_alloc&) { return ehyb::fail_oom(); }              \
  catch (const std::exception& e) { return ehyb::fail(e.what()); }        \
  catch (...) { return ehyb::fail("unknown native error"); }
