// No C++ exception crosses the C ABI (include/pspmm.h, "Errors"): every
// extern "C" entry that returns a pspmm_status runs its body through
// `guarded`, which maps std::bad_alloc / std::length_error (a host container
// sized beyond memory) to PSPMM_ERR_OOM and any other exception to
// PSPMM_ERR_INVALID_ARG, recording the message for pspmm_last_error().
#pragma once

#include <exception>
#include <new>
#include <stdexcept>
#include <string>

#include "pspmm.h"

namespace pspmm {

void set_error(const std::string &msg);  // capi.cu; never throws
void set_error_cstr(const char *where, const char *what) noexcept;

template <typename Fn>
pspmm_status guarded(const char *where, Fn &&fn) noexcept {
  try {
    return fn();
  } catch (const std::bad_alloc &) {
    set_error_cstr(where, "host allocation failed");
    return PSPMM_ERR_OOM;
  } catch (const std::length_error &) {
    set_error_cstr(where, "host allocation larger than the address space");
    return PSPMM_ERR_OOM;
  } catch (const std::exception &e) {
    set_error_cstr(where, e.what());
    return PSPMM_ERR_INVALID_ARG;
  } catch (...) {
    set_error_cstr(where, "unknown C++ exception");
    return PSPMM_ERR_INVALID_ARG;
  }
}

}  // namespace pspmm
