#include "threadpool.hpp"

#include <cstdlib>

namespace asb {
// Size: ASB_STAGING_THREADS, default all hardware threads but one (the
// caller's thread typically waits on the GPU at the same time).
ThreadPool& staging_pool() {
  static ThreadPool pool([] {
    if (const char* e = std::getenv("ASB_STAGING_THREADS")) return (unsigned)std::max(1, std::atoi(e));
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    return hw - 1;
  }());
  return pool;
}
}  // namespace asb
