// Launch counters + opt-in CUDA-event timing per kernel class.
#include <mutex>
#include <vector>
#include "common.cuh"
#include "prof.cuh"

namespace chm {
namespace prof {

namespace {
struct Rec {
  int kind;
  cudaEvent_t a, b;
  double work;
};
std::mutex mu;
bool enabled = false;
long long launches[K_NUM] = {0};
std::vector<Rec> recs;
std::vector<cudaEvent_t> pool;
int open_kind = -1;
cudaEvent_t open_ev = nullptr;

cudaEvent_t get_event() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

void begin(int kind, cudaStream_t s) {
  std::lock_guard<std::mutex> g(mu);
  if (!enabled) return;
  open_kind = kind;
  open_ev = get_event();
  cudaEventRecord(open_ev, s);
}

void end(int kind, cudaStream_t s, double work) {
  std::lock_guard<std::mutex> g(mu);
  launches[kind] += 1;
  if (!enabled || open_kind != kind || !open_ev) return;
  cudaEvent_t b = get_event();
  cudaEventRecord(b, s);
  recs.push_back({kind, open_ev, b, work});
  open_ev = nullptr;
  open_kind = -1;
}

}  // namespace prof
}  // namespace chm

extern "C" chm_status chm_profile_enable(int32_t enable) {
  std::lock_guard<std::mutex> g(chm::prof::mu);
  chm::prof::enabled = enable != 0;
  return CHM_OK;
}

// Synchronises on the recorded events and returns, per kernel class, the number
// of timed launches, their summed duration (ms) and summed algorithmic work;
// clears the timing records. Launch counters (all launches, timed or not)
// are returned in `launches` and are cumulative.
extern "C" chm_status chm_profile_read(int32_t* timed, double* total_ms, double* work,
                                       int64_t* launches) {
  std::lock_guard<std::mutex> g(chm::prof::mu);
  using namespace chm::prof;
  for (int k = 0; k < K_NUM; ++k) {
    if (timed) timed[k] = 0;
    if (total_ms) total_ms[k] = 0;
    if (work) work[k] = 0;
    if (launches) launches[k] = chm::prof::launches[k];
  }
  for (auto& r : recs) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess) return CHM_ERR_CUDA;
    if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) return CHM_ERR_CUDA;
    if (timed) timed[r.kind] += 1;
    if (total_ms) total_ms[r.kind] += ms;
    if (work) work[r.kind] += r.work;
    pool.push_back(r.a);
    pool.push_back(r.b);
  }
  recs.clear();
  return CHM_OK;
}
