// Error convention of the boundary, mirroring include/lsgd/common.hpp:16-47 of the reference.
#pragma once

#include <cstdint>
#include <sstream>
#include <stdexcept>
#include <string>

namespace lsgd_b200 {

constexpr int kMaxPeers = 16;  // max workers per group and groups per world (flag fan-in / fan-out)


class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class ConfigError : public Error {
 public:
  explicit ConfigError(const std::string& what) : Error(what) {}
};
class TransportError : public Error {
 public:
  explicit TransportError(const std::string& what) : Error(what) {}
};

template <typename... Args>
std::string cat(const Args&... args) {
  std::ostringstream os;
  (os << ... << args);
  return os.str();
}

template <typename Err = Error, typename... Args>
void check(bool cond, const Args&... args) {
  if (!cond) throw Err(cat(args...));
}

// Which phase the calling host thread is in, for "rank R in phase P" error tags (executors.cpp:42, 507-509).
const char*& current_phase();
// Thread-local message behind lsgd_b200_last_error().
std::string& last_error_slot();

}  // namespace lsgd_b200

#define LSGD_CUDA(expr)                                                                                \
  do {                                                                                                 \
    cudaError_t e_ = (expr);                                                                           \
    if (e_ != cudaSuccess)                                                                             \
      throw ::lsgd_b200::Error(::lsgd_b200::cat("CUDA error ", cudaGetErrorString(e_), " at ", __FILE__, \
                                                ":", __LINE__, " (", #expr, ")"));                     \
  } while (0)

#define LSGD_NCCL(expr)                                                                                   \
  do {                                                                                                    \
    ncclResult_t r_ = (expr);                                                                             \
    if (r_ != ncclSuccess)                                                                                \
      throw ::lsgd_b200::TransportError(::lsgd_b200::cat("NCCL error ", ncclGetErrorString(r_), " at ",  \
                                                         __FILE__, ":", __LINE__, " (", #expr, ")"));     \
  } while (0)
