// Shared host-side plumbing for the C-ABI: status codes, the thread-local
// error message, and exception types that map 1:1 onto the reference's
// (csr_graph.hpp:12-17, pattern.hpp:49-51, std::invalid_argument).
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>

#include "agpm_b200.h"

namespace agpm_b200 {

struct pattern_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct io_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct parse_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct nodevice_error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& msg);

// Run f, translating exceptions into an AGPM_E* status + message.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return AGPM_OK;
  } catch (const pattern_error& e) {
    set_last_error(e.what());
    return AGPM_E_PATTERN;
  } catch (const io_error& e) {
    set_last_error(e.what());
    return AGPM_E_IO;
  } catch (const parse_error& e) {
    set_last_error(e.what());
    return AGPM_E_PARSE;
  } catch (const std::invalid_argument& e) {
    set_last_error(e.what());
    return AGPM_E_INVALID;
  } catch (const nodevice_error& e) {
    set_last_error(e.what());
    return AGPM_E_NODEVICE;
  } catch (const cuda_error& e) {
    set_last_error(e.what());
    return AGPM_E_CUDA;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return AGPM_E_INTERNAL;
  }
}

// Run `body(begin, end)` over [0, n) on up to hardware_concurrency threads.
void parallel_for(uint64_t n, uint64_t grain, const std::function<void(uint64_t, uint64_t)>& body);

}  // namespace agpm_b200
