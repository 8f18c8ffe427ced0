// NEXT row F4: the control plane above the migration mechanisms (§4.4):
//   Alg. 2  load-aware request scheduling across prefill instances (eqs. 37-38),
//   Alg. 1  adaptive module migration for one control cycle (eqs. 32-36).
// Host-only C++, O(|P| log |P| + |Q| log |P|) dispatch with two ordered sets, O(|D|) per
// migration step.  Readings R-F4a..R-F4g fix what the pseudo-code leaves open;
// the same readings are written out independently in oracle/policy.py.
#include <cmath>
#include <set>
#include <tuple>
#include <vector>

#include "internal.h"

extern "C" {

double bs_utilization(double c, double c_max, double m, double m_max) {
  return c / c_max + m / m_max;  // eq. 32 / eq. 37
}

bs_status bs_dispatch_requests(int32_t n_inst, double* load, int32_t* q_len, int32_t n_req,
                               const double* est_load, double delta_l, int32_t* assign_out) {
  BS_REQUIRE(n_inst >= 1 && n_req >= 0, "bs_dispatch_requests: n_inst %d n_req %d", n_inst, n_req);
  BS_REQUIRE(load && q_len && (n_req == 0 || (est_load && assign_out)),
             "bs_dispatch_requests: NULL argument");
  // least-loaded order (load, q_len, index) and lowest-queue order (q_len, load, index)
  using K1 = std::tuple<double, int32_t, int32_t>;
  using K2 = std::tuple<int32_t, double, int32_t>;
  std::set<K1> by_load;
  std::set<K2> by_queue;
  for (int32_t i = 0; i < n_inst; ++i) {
    by_load.insert(K1{load[i], q_len[i], i});
    by_queue.insert(K2{q_len[i], load[i], i});
  }
  auto update = [&](int32_t i, double new_load, int32_t new_q) {
    by_load.erase(K1{load[i], q_len[i], i});
    by_queue.erase(K2{q_len[i], load[i], i});
    load[i] = new_load;
    q_len[i] = new_q;
    by_load.insert(K1{load[i], q_len[i], i});
    by_queue.insert(K2{q_len[i], load[i], i});
  };
  for (int32_t r = 0; r < n_req; ++r) {
    int32_t target = std::get<2>(*by_load.begin());  // Alg. 2 line 12 (R-F4a)
    if (load[target] < delta_l) {                    // line 13
      update(target, load[target] + est_load[r], q_len[target] + 1);  // lines 14-15, R-F4b
    } else {
      target = std::get<2>(*by_queue.begin());       // lines 16-18 (R-F4c: no load update)
      update(target, load[target], q_len[target] + 1);
    }
    assign_out[r] = target;
  }
  return BS_OK;
}

bs_status bs_plan_migrations(int32_t n_dev, double* load, int32_t* n_layers, const double* layer_load,
                             const double* layer_cost, int32_t* n_heads, const double* head_load,
                             const double* head_cost, const uint8_t* supports_layer,
                             const uint8_t* supports_attn, double delta, double rho,
                             int32_t max_moves, int32_t* moves_out, int32_t* n_moves_out) {
  BS_REQUIRE(n_dev >= 1 && max_moves >= 0, "bs_plan_migrations: n_dev %d", n_dev);
  BS_REQUIRE(load && n_layers && layer_load && layer_cost && n_heads && head_load && head_cost &&
                 supports_layer && supports_attn && n_moves_out && (max_moves == 0 || moves_out),
             "bs_plan_migrations: NULL argument");
  int32_t nm = 0;
  while (nm < max_moves) {
    double lo = load[0], hi = load[0];
    for (int32_t d = 1; d < n_dev; ++d) {
      lo = std::min(lo, load[d]);
      hi = std::max(hi, load[d]);
    }
    // eq. 33 classification; d_o = most loaded overloaded, d_u = least loaded underloaded
    int32_t d_o = -1, d_u = -1;
    for (int32_t d = 0; d < n_dev; ++d)
      if (load[d] - lo > delta && (d_o < 0 || load[d] > load[d_o])) d_o = d;
    bool any_under = false;
    for (int32_t d = 0; d < n_dev; ++d)
      if (hi - load[d] > delta) any_under = true;
    if (d_o < 0 || !any_under) break;
    for (int32_t d = 0; d < n_dev; ++d)
      if (d != d_o && hi - load[d] > delta && (d_u < 0 || load[d] < load[d_u])) d_u = d;
    if (d_u < 0) break;
    const double gap = load[d_o] - load[d_u];  // eq. 34 (R-F4d)
    bool done = false;
    for (int kind = 0; kind < 2 && !done; ++kind) {  // Alg. 1 lines 12-16 (R-F4e)
      if (gap < delta) break;
      if (kind == 0 && !(supports_layer[d_o] && n_layers[d_o] > 0)) continue;
      if (kind == 1 && !(supports_attn[d_o] && n_heads[d_o] > 0)) continue;
      const double u = kind == 0 ? layer_load[d_o] : head_load[d_o];
      const double cost = kind == 0 ? layer_cost[d_o] : head_cost[d_o];
      const double after = std::fabs((load[d_o] - u) - (load[d_u] + u));
      const double benefit = gap - after;  // eq. 35
      if (cost > 0 && benefit / cost >= rho) {
        load[d_o] -= u;  // line 17 (R-F4f)
        load[d_u] += u;
        int32_t* cnt = kind == 0 ? n_layers : n_heads;
        cnt[d_o] -= 1;
        cnt[d_u] += 1;
        moves_out[3 * nm + 0] = kind;
        moves_out[3 * nm + 1] = d_o;
        moves_out[3 * nm + 2] = d_u;
        ++nm;
        done = true;
      }
    }
    if (!done) break;
  }
  *n_moves_out = nm;
  return BS_OK;
}

}  // extern "C"
