// ATP cost model and mesh search, pure host C++ (§3.3-§3.5, §5.4).
//
//   Eq. 3  effective bandwidths B1', B2' from the hierarchical
//                      communication matrix (reading G5/G6 in DESIGN.md)
//   Eq. 4  Rabenseifner: B = d / (2(d-1)) * B'
//   Eq. 2  T = 2Lbs (3h/(d1 B2) + h/(d2 B1) + 4h/(d1 B2) + h/(d2 B1))
//   search argmin over all (d1, d2), d1*d2 = N; ties -> larger d1
//
// Every double is evaluated in the canonical order listed in DESIGN.md
// ("Canonical evaluation order") so results are bit-identical to the oracle.
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/atp.h"

namespace atp {
void set_error(const std::string& msg);

namespace {

struct Spans {
  int k1[ATP_MAX_HCM_LAYERS];
  int k2[ATP_MAX_HCM_LAYERS];
};

// Mesh dim 2 is innermost (rank = i1*d2 + i2): it takes whole inner layers,
// then an even divisor of the next one.  Returns false on misalignment.
bool spans(const atp_hcm& hcm, int d2, Spans& s) {
  int rem = d2;
  for (int j = 0; j < hcm.n_layers; ++j) s.k2[j] = 1;
  for (int j = hcm.n_layers - 1; j >= 0 && rem > 1; --j) {
    const int R = hcm.ranks[j];
    if (rem >= R) {
      if (rem % R) return false;
      s.k2[j] = R;
      rem /= R;
    } else {
      if (R % rem) return false;
      s.k2[j] = rem;
      rem = 1;
    }
  }
  if (rem != 1) return false;
  for (int j = 0; j < hcm.n_layers; ++j) s.k1[j] = hcm.ranks[j] / s.k2[j];
  return true;
}

// B'_j = min(GroupBW_j, (k_j - 1) * P2P_j) / share_j, B' = min over spanned layers.
// Returns 0.0 for NoComm (dimension of size 1).
bool eq3(const atp_hcm& hcm, int d1, int d2, double& b1p, double& b2p) {
  Spans s;
  if (!spans(hcm, d2, s)) return false;
  bool have1 = false, have2 = false;
  b1p = 0.0;
  b2p = 0.0;
  for (int j = 0; j < hcm.n_layers; ++j) {
    long long devs = 1;  // devices inside one layer-j rank
    for (int jj = j + 1; jj < hcm.n_layers; ++jj) devs *= hcm.ranks[jj];
    if (s.k1[j] > 1) {
      const double cap = static_cast<double>(s.k1[j] - 1) * hcm.p2p_gbps[j];
      const double g = hcm.group_gbps[j];
      const double m = cap < g ? cap : g;
      const long long share = std::min<long long>(d2, devs);
      const double v = m / static_cast<double>(share);
      if (!have1 || v < b1p) b1p = v;
      have1 = true;
    }
    if (s.k2[j] > 1) {
      const double cap = static_cast<double>(s.k2[j] - 1) * hcm.p2p_gbps[j];
      const double g = hcm.group_gbps[j];
      const double v = (cap < g ? cap : g) / 1.0;
      if (!have2 || v < b2p) b2p = v;
      have2 = true;
    }
  }
  if (d1 == 1) b1p = 0.0;
  if (d2 == 1) b2p = 0.0;
  return true;
}

double eq4(double bp, int d) {
  if (d == 1 || bp <= 0.0) return 0.0;
  return (static_cast<double>(d) * bp) / (2.0 * static_cast<double>(d - 1));
}

void eq2(const atp_model& m, int d1, int d2, double b1, double b2, atp_cost& c) {
  const double h = static_cast<double>(m.h);
  const double t1 = b2 > 0.0 ? (3.0 * h) / (static_cast<double>(d1) * (b2 * 1e9)) : 0.0;
  const double t2 = b1 > 0.0 ? h / (static_cast<double>(d2) * (b1 * 1e9)) : 0.0;
  const double t3 = b2 > 0.0 ? (4.0 * h) / (static_cast<double>(d1) * (b2 * 1e9)) : 0.0;
  const double t4 = b1 > 0.0 ? h / (static_cast<double>(d2) * (b1 * 1e9)) : 0.0;
  const double scale = 2.0 * static_cast<double>(m.L) * static_cast<double>(m.b) * static_cast<double>(m.s) *
                       static_cast<double>(m.bytes_per_elem);
  c.t_f[0] = scale * t1;
  c.t_f[1] = scale * t2;
  c.t_f[2] = scale * t3;
  c.t_f[3] = scale * t4;
  c.t_comm = scale * (((t1 + t2) + t3) + t4);
}

bool valid_hcm(const atp_hcm* hcm, long long* n) {
  if (hcm == nullptr || hcm->n_layers < 1 || hcm->n_layers > ATP_MAX_HCM_LAYERS) return false;
  long long p = 1;
  for (int j = 0; j < hcm->n_layers; ++j) {
    if (hcm->ranks[j] < 1 || !(hcm->p2p_gbps[j] > 0.0) || !(hcm->group_gbps[j] > 0.0)) return false;
    p *= hcm->ranks[j];
  }
  *n = p;
  return true;
}

const char* model_reject(const atp_model& m, int d1, int d2) {
  if (m.h % d2) return "h % d2";
  if (m.h % d1) return "h % d1";
  if (m.heads % d1) return "heads % d1";
  if (m.h % m.heads) return "h % heads";
  return nullptr;
}

}  // namespace
}  // namespace atp

extern "C" {

atp_status atp_effective_bandwidth(const atp_hcm* hcm, int d1, int d2, double* b1p, double* b2p) {
  long long n = 0;
  if (!atp::valid_hcm(hcm, &n) || d1 < 1 || d2 < 1 || b1p == nullptr || b2p == nullptr) {
    atp::set_error("atp_effective_bandwidth: invalid HCM or arguments");
    return ATP_ERR_INVALID;
  }
  if (static_cast<long long>(d1) * d2 != n) {
    atp::set_error("atp_effective_bandwidth: d1*d2 != HCM device count");
    return ATP_ERR_INVALID;
  }
  if (!atp::eq3(*hcm, d1, d2, *b1p, *b2p)) {
    atp::set_error("atp_effective_bandwidth: mesh dim 2 does not align with the HCM layers");
    return ATP_ERR_SHAPE;
  }
  return ATP_OK;
}

atp_status atp_search(const atp_hcm* hcm, const atp_model* model, int n_devices, const atp_calib* calib,
                      atp_plan* out) {
  long long n = 0;
  if (!atp::valid_hcm(hcm, &n) || model == nullptr || out == nullptr) {
    atp::set_error("atp_search: invalid HCM (layers 1..8, ranks >= 1, bandwidths > 0) or NULL argument");
    return ATP_ERR_INVALID;
  }
  if (n != n_devices) {
    atp::set_error("atp_search: product of HCM ranks != n_devices");
    return ATP_ERR_INVALID;
  }
  if (model->L < 1 || model->b < 1 || model->s < 1 || model->h < 1 || model->heads < 1 || model->bytes_per_elem < 1) {
    atp::set_error("atp_search: model fields must be positive");
    return ATP_ERR_INVALID;
  }
  *out = atp_plan{};
  std::vector<atp_cost> reps;
  for (int d1 = n_devices; d1 >= 1; --d1) {
    if (n_devices % d1) continue;
    const int d2 = n_devices / d1;
    if (atp::model_reject(*model, d1, d2)) {
      if (out->n_rejected < ATP_MAX_PLAN) {
        out->rejected_d1[out->n_rejected] = d1;
        out->rejected_d2[out->n_rejected] = d2;
        ++out->n_rejected;
      }
      continue;
    }
    atp_cost c{};
    c.d1 = d1;
    c.d2 = d2;
    int cal = -1;
    if (calib != nullptr)
      for (int i = 0; i < calib->n && i < ATP_MAX_PLAN; ++i)
        if (calib->d1[i] == d1 && calib->d2[i] == d2) cal = i;
    if (cal >= 0) {
      if ((d1 > 1 && !(calib->b1[cal] > 0.0)) || (d2 > 1 && !(calib->b2[cal] > 0.0))) {
        atp::set_error("atp_search: calibration entry lacks a bandwidth for a dimension of size > 1");
        return ATP_ERR_INVALID;
      }
      c.b1 = d1 > 1 ? calib->b1[cal] : 0.0;
      c.b2 = d2 > 1 ? calib->b2[cal] : 0.0;
      c.calibrated = 1;
    } else {
      if (!atp::eq3(*hcm, d1, d2, c.b1_prime, c.b2_prime)) {
        if (out->n_rejected < ATP_MAX_PLAN) {
          out->rejected_d1[out->n_rejected] = d1;
          out->rejected_d2[out->n_rejected] = d2;
          ++out->n_rejected;
        }
        continue;
      }
      c.b1 = atp::eq4(c.b1_prime, d1);
      c.b2 = atp::eq4(c.b2_prime, d2);
    }
    atp::eq2(*model, d1, d2, c.b1, c.b2, c);
    reps.push_back(c);
  }
  if (reps.empty()) {
    atp::set_error("atp_search: no admissible mesh");
    return ATP_ERR_EMPTY;
  }
  std::stable_sort(reps.begin(), reps.end(), [](const atp_cost& a, const atp_cost& b) { return a.t_comm < b.t_comm; });
  out->n_ranked = static_cast<int>(std::min<size_t>(reps.size(), ATP_MAX_PLAN));
  for (int i = 0; i < out->n_ranked; ++i) out->ranked[i] = reps[i];
  out->chosen = 0;
  return ATP_OK;
}

atp_status atp_comm_volume(int d1, int d2, int64_t T, int64_t h, int64_t F, int chunks, atp_call* calls, int cap,
                           int* n_calls, int64_t* dim1_elems, int64_t* dim2_elems) {
  if (d1 < 1 || d2 < 1 || T < 1 || h < 1 || F < 1 || chunks < 1 || n_calls == nullptr) {
    atp::set_error("atp_comm_volume: invalid arguments");
    return ATP_ERR_INVALID;
  }
  if (T % chunks || h % d1 || h % d2 || F % d1) {
    atp::set_error("atp_comm_volume: T % chunks, h % d1, h % d2 and F % d1 must be 0");
    return ATP_ERR_SHAPE;
  }
  const int64_t M = T / chunks;
  // (phase, block, dim, width): the schedule order of the layer (reading G4)
  const struct {
    int phase, block, dim;
    int64_t width;
  } seq[8] = {{0, 0, 2, 3 * h / d1}, {0, 1, 1, h / d2}, {0, 2, 2, F / d1}, {0, 3, 1, h / d2},
              {1, 3, 2, F / d1},     {1, 2, 1, h / d2}, {1, 1, 2, h / d1}, {1, 0, 1, h / d2}};
  int cnt = 0;
  int64_t e1 = 0, e2 = 0;
  for (const auto& st : seq) {
    const int p = st.dim == 1 ? d1 : d2;
    if (p == 1) continue;
    for (int k = 0; k < chunks; ++k) {
      if (calls != nullptr && cnt < cap) calls[cnt] = atp_call{st.phase, st.block, st.dim, p, M * st.width};
      ++cnt;
      (st.dim == 1 ? e1 : e2) += M * st.width;
    }
  }
  *n_calls = cnt;
  if (dim1_elems) *dim1_elems = e1;
  if (dim2_elems) *dim2_elems = e2;
  return ATP_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- overlap model
// Event simulation of the chunk pipeline (§4.1 Fig. 7, §4.2), the same
// max/plus operations in the same order as oracle/overlap.py.
extern "C" atp_status atp_overlap_estimate(int n_stages, const double* comp, const double* dw, const double* comm,
                                           int chunks, int mode, double* makespan, double* exposed) {
  if (n_stages < 0 || chunks < 1 || (mode != 0 && mode != 1) || makespan == nullptr ||
      (n_stages > 0 && (comp == nullptr || dw == nullptr || comm == nullptr))) {
    atp::set_error("atp_overlap_estimate: invalid arguments");
    return ATP_ERR_INVALID;
  }
  const int c = chunks;
  std::vector<double> prev(c, 0.0), cend(c, 0.0);
  double t_cmp = 0.0, t_com = 0.0, total = 0.0;
  for (int s = 0; s < n_stages; ++s) {
    const double gk = comp[s] / c, ak = comm[s] / c;
    if (mode == 0) {
      const double start = t_cmp > prev[c - 1] ? t_cmp : prev[c - 1];
      for (int k = 0; k < c; ++k) cend[k] = start + (k + 1) * gk;
      t_cmp = cend[c - 1];
    } else {
      for (int k = 0; k < c; ++k) {
        const double start = t_cmp > prev[k] ? t_cmp : prev[k];
        cend[k] = start + gk;
        t_cmp = cend[k];
      }
    }
    t_cmp = t_cmp + dw[s];
    for (int k = 0; k < c; ++k) {
      if (comm[s] > 0.0) {
        const double start = t_com > cend[k] ? t_com : cend[k];
        t_com = start + ak;
        prev[k] = t_com;
      } else {
        prev[k] = cend[k];
      }
    }
    total += comp[s] + dw[s];
  }
  const double mk = t_cmp > t_com ? t_cmp : t_com;
  *makespan = mk;
  if (exposed) *exposed = mk - total;
  return ATP_OK;
}

// ---------------------------------------------------------------- chunk planner
// Stage decomposition of one layer fwd+bwd (reading G36) and the
// argmin over candidate chunk counts; same operations in the same order as
// oracle/overlap.py layer_stages / plan_chunks.
namespace {
bool layer_dims_ok(int d1, int d2, int64_t T, int64_t h, int64_t F) {
  return d1 >= 1 && d2 >= 1 && T > 0 && h > 0 && F > 0 && h % d1 == 0 && h % d2 == 0 && (3 * h) % d1 == 0 &&
         F % d1 == 0;
}

void stages8(int d1, int d2, int64_t T, int64_t h, int64_t F, int bytes, double compute_ms, double busbw,
             double* comp, double* dw, double* comm) {
  const int64_t hc = h / d2, h1 = h / d1, q1 = 3 * h / d1, F1 = F / d1;
  struct St { int64_t n, k; bool dw; int dim; int64_t width; };
  const St st[8] = {{q1, hc, false, 2, q1}, {hc, h1, false, 1, hc}, {F1, hc, false, 2, F1}, {hc, F1, false, 1, hc},
                    {F1, hc, true, 2, F1},  {hc, F1, true, 1, hc},  {h1, hc, true, 2, h1},  {hc, q1, true, 1, hc}};
  double g[8], w[8], tot = 0.0;
  for (int i = 0; i < 8; ++i) {
    g[i] = 2.0 * (double)T * (double)st[i].n * (double)st[i].k;
    w[i] = st[i].dw ? 2.0 * (double)st[i].n * (double)st[i].k * (double)T : 0.0;
  }
  for (int i = 0; i < 8; ++i) tot = tot + (g[i] + w[i]);
  for (int i = 0; i < 8; ++i) {
    const int p = st[i].dim == 1 ? d1 : d2;
    const int64_t elems = T * st[i].width;
    comm[i] = p > 1 ? (2.0 * (p - 1) / p * (double)elems * (double)bytes) / (busbw * 1e9) * 1e3 : 0.0;
    comp[i] = compute_ms * g[i] / tot;
    dw[i] = compute_ms * w[i] / tot;
  }
}
}  // namespace

extern "C" atp_status atp_layer_stages(int d1, int d2, int64_t T, int64_t h, int64_t F, int bytes_per_elem,
                                       double compute_ms, double busbw_gbps, double* comp, double* dw,
                                       double* comm) {
  if (!layer_dims_ok(d1, d2, T, h, F) || bytes_per_elem < 1 || !(compute_ms >= 0.0) || !(busbw_gbps > 0.0) ||
      comp == nullptr || dw == nullptr || comm == nullptr) {
    atp::set_error("atp_layer_stages: invalid arguments");
    return ATP_ERR_INVALID;
  }
  stages8(d1, d2, T, h, F, bytes_per_elem, compute_ms, busbw_gbps, comp, dw, comm);
  return ATP_OK;
}

extern "C" atp_status atp_plan_chunks(int d1, int d2, int64_t T, int64_t h, int64_t F, int bytes_per_elem,
                                      int n_cand, const int* chunks, const double* compute_ms, double busbw_gbps,
                                      int mode, int* chosen, double* makespan_ms, double* exposed_ms) {
  if (!layer_dims_ok(d1, d2, T, h, F) || bytes_per_elem < 1 || n_cand < 1 || chunks == nullptr ||
      compute_ms == nullptr || !(busbw_gbps > 0.0) || (mode != 0 && mode != 1) || chosen == nullptr) {
    atp::set_error("atp_plan_chunks: invalid arguments");
    return ATP_ERR_INVALID;
  }
  for (int i = 0; i < n_cand; ++i) {
    if (chunks[i] < 1 || T % chunks[i] || !(compute_ms[i] >= 0.0) || (i > 0 && chunks[i] <= chunks[i - 1])) {
      atp::set_error("atp_plan_chunks: candidates must be ascending chunk counts dividing T with compute >= 0");
      return ATP_ERR_INVALID;
    }
  }
  int best = -1;
  double best_mk = 0.0;
  for (int i = 0; i < n_cand; ++i) {
    double comp[8], dw[8], comm[8], mk = 0.0, ex = 0.0;
    stages8(d1, d2, T, h, F, bytes_per_elem, compute_ms[i], busbw_gbps, comp, dw, comm);
    const atp_status st = atp_overlap_estimate(8, comp, dw, comm, chunks[i], mode, &mk, &ex);
    if (st != ATP_OK) return st;
    if (makespan_ms) makespan_ms[i] = mk;
    if (exposed_ms) exposed_ms[i] = ex;
    if (best < 0 || mk < best_mk) {
      best = i;
      best_mk = mk;
    }
  }
  *chosen = chunks[best];
  return ATP_OK;
}
