// Host-side native runtime pieces: error reporting, device query, ILU(0)
// factorisation and level scheduling of the 1D block.
//
// Compiled with -ffp-contract=off so the factorisation performs exactly the
// reference's rounded operations (krylov.py:188-216) and the factor -- hence
// the device sweeps -- matches the reference bitwise.
#include <stdlib.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <vector>

#include "../../include/mdp_b200.h"

namespace mdp {

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    // opt-in: inside the solve's CUDA graphs PDL measured +0.6% at 33^3 but
    // eager 129^3 CNN forwards lost 10% (profiles/r01_pdl_ab.txt)
    const char* e = getenv("MDP_PDL");
    on = e ? atoi(e) != 0 : 0;
  }
  return on != 0;
}

int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      cached = v;
    else
      cached = 148;
  }
  return cached;
}

}  // namespace mdp

extern "C" const char* mdp_last_error(void) { return mdp::g_err; }

extern "C" int mdp_version(void) { return 1; }

extern "C" long long mdp_launch_count(void) { return mdp::g_launches.load(); }

extern "C" int mdp_device_sm_count(void) { return mdp::sm_count(); }

static const double kBreakdownTol = 1e-14;  // krylov.py:28

extern "C" int64_t mdp_ilu0_factor_host(int64_t n, const int64_t* ip, const int64_t* ix, double* a,
                                        const int64_t* dp) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t p = ip[i];
    while (p < ip[i + 1] && ix[p] < i) {
      const int64_t k = ix[p];
      const double piv = a[dp[k]];
      if (fabs(piv) < kBreakdownTol) return k;
      const double lik = a[p] / piv;
      a[p] = lik;
      int64_t pk = dp[k] + 1, pi = p + 1;
      while (pk < ip[k + 1] && pi < ip[i + 1]) {
        const int64_t ck = ix[pk], ci = ix[pi];
        if (ck == ci) {
          const double prod = lik * a[pk];
          a[pi] = a[pi] - prod;
          ++pk;
          ++pi;
        } else if (ck < ci) {
          ++pk;
        } else {
          ++pi;
        }
      }
      ++p;
    }
    if (fabs(a[dp[i]]) < kBreakdownTol) return i;
  }
  return -1;
}

extern "C" int mdp_ilu0_levels_host(int64_t n, const int64_t* ip, const int64_t* ix, const int64_t* dp,
                                    int32_t* perm_f, int32_t* lev_f, int32_t* nlev_f, int32_t* perm_b,
                                    int32_t* lev_b, int32_t* nlev_b) {
  std::vector<int32_t> lf(n, 0), lb(n, 0);
  int32_t mf = 0, mb = 0;
  for (int64_t i = 0; i < n; ++i) {  // forward: depends on earlier rows in L
    int32_t l = 0;
    for (int64_t p = ip[i]; p < dp[i]; ++p) l = std::max(l, lf[ix[p]] + 1);
    lf[i] = l;
    mf = std::max(mf, l + 1);
  }
  for (int64_t i = n - 1; i >= 0; --i) {  // backward: depends on later rows in U
    int32_t l = 0;
    for (int64_t p = dp[i] + 1; p < ip[i + 1]; ++p) l = std::max(l, lb[ix[p]] + 1);
    lb[i] = l;
    mb = std::max(mb, l + 1);
  }
  auto bucket = [n](const std::vector<int32_t>& lev, int32_t m, int32_t* perm, int32_t* bounds) {
    std::vector<int32_t> cnt(m + 1, 0);
    for (int64_t i = 0; i < n; ++i) cnt[lev[i] + 1]++;
    for (int32_t L = 0; L < m; ++L) cnt[L + 1] += cnt[L];
    for (int32_t L = 0; L <= m; ++L) bounds[L] = cnt[L];
    std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
    for (int64_t i = 0; i < n; ++i) perm[pos[lev[i]]++] = (int32_t)i;
  };
  if (n == 0) {
    mf = mb = 0;
    lev_f[0] = lev_b[0] = 0;
  } else {
    bucket(lf, mf, perm_f, lev_f);
    bucket(lb, mb, perm_b, lev_b);
  }
  *nlev_f = mf;
  *nlev_b = mb;
  return 0;
}
