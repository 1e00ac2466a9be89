// capi_common.hpp — status/exception mapping shared by the host and device
// halves of the C-ABI (SURVEY.md 8(b) "Error conventions").
#pragma once

#include <stdexcept>
#include <string>

#include "lg.h"

namespace lgc {

void set_error(const std::string& msg);

struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <typename F>
int guard(F&& f) {
  try {
    f();
    return LG_OK;
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return LG_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    set_error(e.what());
    return LG_ERR_OUT_OF_RANGE;
  } catch (const cuda_error& e) {
    set_error(e.what());
    return LG_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    set_error("out of memory");
    return LG_ERR_NOMEM;
  } catch (const std::exception& e) {
    set_error(e.what());
    return LG_ERR_RUNTIME;
  }
}

}  // namespace lgc
