#include "threadpool.hpp"

namespace asb {
ThreadPool& staging_pool() {
  static ThreadPool pool;
  return pool;
}
}  // namespace asb
