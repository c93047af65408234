// Stale-statistics scheduler (Algorithms 1-2), host logic restated from
// include/spngd/stale.hpp:56-132.  The similarity norms it consumes are
// computed on the device by K8 (precond.cu: stat_distance_kernel) on the
// owner's reduced statistic and its two retained snapshots.
#include <algorithm>
#include <string>

#include "spngd_b200.h"

struct spngd_tracker {
  std::string id;
  double alpha = 0.1;
  int64_t t_x = 1, delta = 1, delta_prev = 1, refresh_count = 0;  // stale.hpp:126-130
  int snapshots = 0;  // how many of x1, x2 exist
};

namespace spngd {
int fail(int code, const char* fmt, ...);
}

namespace {
// similar(): ||x - ref|| / ||ref|| < alpha; zero reference only matches exactly (stale.hpp:56-64).
bool similar(double dn, double rn, double alpha) {
  if (rn == 0.0) return dn == 0.0;
  return dn / rn < alpha;
}
}  // namespace

extern "C" {

spngd_tracker* spngd_tracker_create(const char* id, double alpha) {
  auto* t = new spngd_tracker();
  t->id = id ? id : "";
  t->alpha = alpha;
  return t;
}

void spngd_tracker_destroy(spngd_tracker* t) { delete t; }

int spngd_tracker_should_refresh(const spngd_tracker* t, int64_t step) { return t && step == t->t_x; }  // stale.hpp:98

int spngd_tracker_on_refresh(spngd_tracker* t, int64_t step, int has1, double d1, double r1, int has2, double d2,
                             double r2, int64_t* next_interval, int* reason) {
  if (!t) return spngd::fail(SPNGD_ERR_INVALID, "tracker is NULL");
  if (step != t->t_x)
    return spngd::fail(SPNGD_ERR_REFRESH_OUT_OF_TURN, "statistic %s: refresh at step %lld but scheduled for %lld",
                       t->id.c_str(), (long long)step, (long long)t->t_x);
  // next_interval (stale.hpp:78-88); absent snapshots count as dissimilar.
  int64_t nd;
  int why;
  if (!has1) {
    nd = std::max<int64_t>(1, t->delta / 2);
    why = 0;
  } else if (!similar(d1, r1, t->alpha)) {
    nd = std::max<int64_t>(1, t->delta / 2);
    why = 1;
  } else if (!has2 || !similar(d2, r2, t->alpha)) {
    nd = t->delta;
    why = 2;
  } else {
    nd = t->delta + t->delta_prev;
    why = 3;
  }
  // Snapshot rotation is the caller's (device buffers); bookkeeping here.
  t->snapshots = std::min(2, t->snapshots + 1);
  t->delta_prev = t->delta;
  t->delta = nd;
  t->t_x = step + nd;
  ++t->refresh_count;
  if (next_interval) *next_interval = nd;
  if (reason) *reason = why;
  return SPNGD_OK;
}

void spngd_tracker_state(const spngd_tracker* t, int64_t* t_x, int64_t* delta, int64_t* delta_prev,
                         int64_t* refresh_count) {
  if (!t) return;
  if (t_x) *t_x = t->t_x;
  if (delta) *delta = t->delta;
  if (delta_prev) *delta_prev = t->delta_prev;
  if (refresh_count) *refresh_count = t->refresh_count;
}

}  // extern "C"
