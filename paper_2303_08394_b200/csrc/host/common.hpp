// Shared host types, the error taxonomy and the C-ABI status plumbing.
//
// The exception classes mirror the reference taxonomy one-for-one
// (proj/src/common.hpp:19-49); DeviceError is new and covers CUDA / NCCL.
// Exceptions never cross the C ABI: `guard()` converts them to kifmm_status
// and stores the message in a thread-local slot (kifmm_last_error()).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "kifmm.h"

namespace kifmm {

class InvalidArgument : public std::invalid_argument {  // common.hpp:21
 public:
  using std::invalid_argument::invalid_argument;
};
class IoError : public std::runtime_error {  // common.hpp:27
 public:
  using std::runtime_error::runtime_error;
};
class NumericalError : public std::runtime_error {  // common.hpp:33
 public:
  using std::runtime_error::runtime_error;
};
class CacheMismatch : public std::runtime_error {  // common.hpp:40
 public:
  using std::runtime_error::runtime_error;
};
class CorruptArchive : public std::runtime_error {  // common.hpp:46
 public:
  using std::runtime_error::runtime_error;
};
class DeviceError : public std::runtime_error {  // new: CUDA failures
 public:
  DeviceError(kifmm_status s, const std::string& m) : std::runtime_error(m), status(s) {}
  kifmm_status status;
};

void set_last_error(const std::string& msg);
void clear_last_error();

// Runs `f`, mapping exceptions to status codes.
template <class F>
kifmm_status guard(F&& f) {
  try {
    clear_last_error();
    f();
    return KIFMM_OK;
  } catch (const InvalidArgument& e) {
    set_last_error(e.what());
    return KIFMM_E_INVALID_ARGUMENT;
  } catch (const IoError& e) {
    set_last_error(e.what());
    return KIFMM_E_IO;
  } catch (const NumericalError& e) {
    set_last_error(e.what());
    return KIFMM_E_NUMERICAL;
  } catch (const CacheMismatch& e) {
    set_last_error(e.what());
    return KIFMM_E_CACHE_MISMATCH;
  } catch (const CorruptArchive& e) {
    set_last_error(e.what());
    return KIFMM_E_CORRUPT_ARCHIVE;
  } catch (const DeviceError& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return KIFMM_E_OUT_OF_MEMORY;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return KIFMM_E_INTERNAL;
  } catch (...) {
    set_last_error("unknown error");
    return KIFMM_E_INTERNAL;
  }
}

constexpr double kPi = 3.14159265358979323846;
constexpr double kInv4Pi = 1.0 / (4.0 * kPi);

// SPEC.md:294-302.  1/(4 pi r), exactly 0 at r = 0.
inline double laplace(double x0, double x1, double x2, double y0, double y1, double y2) {
  const double dx = x0 - y0, dy = x1 - y1, dz = x2 - y2;
  const double r2 = dx * dx + dy * dy + dz * dz;
  if (r2 == 0.0) return 0.0;
  return kInv4Pi / std::sqrt(r2);
}

}  // namespace kifmm
