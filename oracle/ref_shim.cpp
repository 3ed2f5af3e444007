// TEST INFRASTRUCTURE ONLY — a C-ABI shim over the UNMODIFIED reference
// headers (nttkit, /root/reference/proj/include/nttkit/*.hpp), compiled by
// oracle/Makefile into oracle/_ref/libnttref.so. No reference source is copied
// into this repository: the headers are included from where they lie.
//
// Used (1) to pin the C oracle (oracle/nttkit_oracle.c) against the reference
// itself, (2) to generate tests/golden/ fixtures, and (3) as the CPU baseline
// (`cpu_baseline.kind = "reference"`) and `bench.py --impl reference` arm,
// running the reference's own NttTables::forward/inverse, eltwise_mult_mod,
// eltwise_fma_mod and poly_mult_mod over independent rows on all host threads
// (tables are immutable and shareable, ntt.hpp:203-205).
#include <pthread.h>
#include <sched.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "nttkit/eltwise.hpp"
#include "nttkit/modarith.hpp"
#include "nttkit/ntt.hpp"
#include "nttkit/ring.hpp"

using namespace nttkit;

namespace {

thread_local char g_err[256];

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    std::strncpy(g_err, e.what(), sizeof(g_err) - 1);
    return -1;
  }
}

std::vector<std::unique_ptr<NttTables>> make_tables(uint64_t n, const uint64_t* moduli,
                                                    uint32_t nmod, int bit_shift) {
  std::vector<std::unique_ptr<NttTables>> t;
  for (uint32_t i = 0; i < nmod; ++i) {
    Modulus m(moduli[i]);
    if (bit_shift == 0)
      t.emplace_back(std::make_unique<NttTables>(n, m));
    else
      t.emplace_back(std::make_unique<NttTables>(n, m, std::nullopt, bit_shift));
  }
  return t;
}

// CPUs the workers are placed on: the process's affinity mask when the shim
// is first used (captured once, so nothing that later narrows the calling
// thread's mask can collapse the placement)
const std::vector<int>& worker_cpus() {
  static const std::vector<int> cpus = [] {
    std::vector<int> v;
    const char* e = std::getenv("NK_REF_PIN");
    if (e && e[0] == '0') return v;
    cpu_set_t allowed;
    CPU_ZERO(&allowed);
    if (sched_getaffinity(0, sizeof(allowed), &allowed) == 0)
      for (int c = 0; c < CPU_SETSIZE; ++c)
        if (CPU_ISSET(c, &allowed)) v.push_back(c);
    return v;
  }();
  return cpus;
}

template <class F>
void parallel_rows(uint64_t rows, int threads, F&& body) {
  if (threads <= 1 || rows <= 1) {
    for (uint64_t r = 0; r < rows; ++r) body(r);
    return;
  }
  if ((uint64_t)threads > rows) threads = (int)rows;
  // fixed placement: worker t on the t-th allowed CPU, so repeated
  // measurements see the same thread-to-core mapping. Each worker pins
  // itself: pinning it from here through its handle races with its exit
  // (an exited thread's handle resolves to the caller, which would pin the
  // calling thread instead).
  const std::vector<int>& cpus = worker_cpus();
  std::vector<std::thread> pool;
  pool.reserve(threads);
  for (int t = 0; t < threads; ++t) {
    const uint64_t r0 = rows * t / threads, r1 = rows * (t + 1) / threads;
    const int cpu = cpus.empty() ? -1 : cpus[t % cpus.size()];
    pool.emplace_back([&body, r0, r1, cpu] {
      if (cpu >= 0) {
        cpu_set_t one;
        CPU_ZERO(&one);
        CPU_SET(cpu, &one);
        pthread_setaffinity_np(pthread_self(), sizeof(one), &one);
      }
      for (uint64_t r = r0; r < r1; ++r) body(r);
    });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err; }

int ref_hw_threads() { return (int)std::thread::hardware_concurrency(); }

int ref_tables(uint64_t n, uint64_t q, uint64_t root, int bit_shift, uint64_t* psi,
               uint64_t* w, uint64_t* wp, uint64_t* wi, uint64_t* wip, uint64_t* ninv,
               uint64_t* ninvp, int* bs_out) {
  return guarded([&] {
    Modulus m(q);
    std::optional<uint64_t> r;
    if (root) r = root;
    int bs = bit_shift;
    if (bs == 0) bs = 4 * static_cast<uint128_t>(q) < (uint128_t{1} << 52) ? 52 : 64;
    NttTables t(n, m, r, bs);
    if (psi) *psi = t.root();
    if (w) std::memcpy(w, t.root_powers_rev().data(), n * 8);
    if (wp) std::memcpy(wp, t.root_precons_rev().data(), n * 8);
    if (wi) std::memcpy(wi, t.inv_root_powers_rev().data(), n * 8);
    if (wip) std::memcpy(wip, t.inv_root_precons_rev().data(), n * 8);
    if (ninv) *ninv = t.inv_size().operand;
    if (ninvp) *ninvp = t.inv_size().precon;
    if (bs_out) *bs_out = t.bit_shift();
  });
}

// Batch of `rows` contiguous length-n rows; row r uses moduli[r % nmod].
int ref_ntt_forward(uint64_t n, const uint64_t* moduli, uint32_t nmod, int bit_shift,
                    uint64_t* res, const uint64_t* op, uint64_t rows, uint64_t fin,
                    uint64_t fout, int threads) {
  return guarded([&] {
    auto t = make_tables(n, moduli, nmod, bit_shift);
    parallel_rows(rows, threads, [&](uint64_t r) {
      t[r % nmod]->forward(std::span<uint64_t>(res + r * n, n),
                           std::span<const uint64_t>(op + r * n, n), fin, fout);
    });
  });
}

int ref_ntt_inverse(uint64_t n, const uint64_t* moduli, uint32_t nmod, int bit_shift,
                    uint64_t* res, const uint64_t* op, uint64_t rows, uint64_t fin,
                    uint64_t fout, int threads) {
  return guarded([&] {
    auto t = make_tables(n, moduli, nmod, bit_shift);
    parallel_rows(rows, threads, [&](uint64_t r) {
      t[r % nmod]->inverse(std::span<uint64_t>(res + r * n, n),
                           std::span<const uint64_t>(op + r * n, n), fin, fout);
    });
  });
}

// Tables built once and reused across calls (bench loop: table construction is
// outside the timed region, as in bench.hpp:252-255).
void* ref_plan_create(uint64_t n, const uint64_t* moduli, uint32_t nmod) {
  try {
    return new std::vector<std::unique_ptr<NttTables>>(make_tables(n, moduli, nmod, 0));
  } catch (const std::invalid_argument& e) {
    std::strncpy(g_err, e.what(), sizeof(g_err) - 1);
    return nullptr;
  }
}
void ref_plan_destroy(void* p) { delete static_cast<std::vector<std::unique_ptr<NttTables>>*>(p); }

int ref_plan_ntt(void* p, int dir, uint64_t* res, const uint64_t* op, uint64_t rows,
                 uint64_t fin, uint64_t fout, int threads) {
  auto& t = *static_cast<std::vector<std::unique_ptr<NttTables>>*>(p);
  const uint64_t n = t[0]->size();
  const uint64_t nmod = t.size();
  return guarded([&] {
    parallel_rows(rows, threads, [&](uint64_t r) {
      std::span<uint64_t> out(res + r * n, n);
      std::span<const uint64_t> in(op + r * n, n);
      if (dir == 0) t[r % nmod]->forward(out, in, fin, fout);
      else t[r % nmod]->inverse(out, in, fin, fout);
    });
  });
}

int ref_plan_poly_mult(void* p, uint64_t* res, const uint64_t* f, const uint64_t* g,
                       uint64_t rows, int threads) {
  auto& t = *static_cast<std::vector<std::unique_ptr<NttTables>>*>(p);
  const uint64_t n = t[0]->size();
  const uint64_t nmod = t.size();
  return guarded([&] {
    parallel_rows(rows, threads, [&](uint64_t r) {
      poly_mult_mod(std::span<uint64_t>(res + r * n, n), std::span<const uint64_t>(f + r * n, n),
                    std::span<const uint64_t>(g + r * n, n), *t[r % nmod]);
    });
  });
}

// path: 0 = the reference's dispatch, 1 = integer path, 2 = float path
int ref_eltwise_mult_mod(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t n,
                         uint64_t q, uint64_t fin, int path, int threads) {
  return guarded([&] {
    Modulus m(q);
    const uint64_t chunks = threads > 1 ? (uint64_t)threads : 1;
    parallel_rows(chunks, threads, [&](uint64_t c) {
      const uint64_t i0 = n * c / chunks, i1 = n * (c + 1) / chunks;
      std::span<uint64_t> rs(r + i0, i1 - i0);
      std::span<const uint64_t> as(a + i0, i1 - i0), bs(b + i0, i1 - i0);
      if (path == 1) eltwise_mult_mod_int(rs, as, bs, m, fin);
      else if (path == 2) eltwise_mult_mod_float(rs, as, bs, m, fin);
      else eltwise_mult_mod(rs, as, bs, m, fin);
    });
  });
}

int ref_eltwise_fma_mod(uint64_t* r, const uint64_t* a, uint64_t y, const uint64_t* z,
                        uint64_t n, uint64_t q, uint64_t fin, int bit_shift, int threads) {
  return guarded([&] {
    Modulus m(q);
    const uint64_t chunks = threads > 1 ? (uint64_t)threads : 1;
    parallel_rows(chunks, threads, [&](uint64_t c) {
      const uint64_t i0 = n * c / chunks, i1 = n * (c + 1) / chunks;
      std::span<uint64_t> rs(r + i0, i1 - i0);
      std::span<const uint64_t> as(a + i0, i1 - i0);
      std::optional<std::span<const uint64_t>> zs;
      if (z) zs = std::span<const uint64_t>(z + i0, i1 - i0);
      if (bit_shift == 52) eltwise_fma_mod<52>(rs, as, y, zs, m, fin);
      else if (bit_shift == 64) eltwise_fma_mod<64>(rs, as, y, zs, m, fin);
      else eltwise_fma_mod(rs, as, y, zs, m, fin);
    });
  });
}

int ref_eltwise_add_mod(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q) {
  return guarded([&] {
    eltwise_add_mod(std::span<uint64_t>(r, n), std::span<const uint64_t>(a, n),
                    std::span<const uint64_t>(b, n), Modulus(q));
  });
}

int ref_eltwise_neg_mod(uint64_t* r, const uint64_t* a, uint64_t n, uint64_t q) {
  return guarded([&] {
    eltwise_neg_mod(std::span<uint64_t>(r, n), std::span<const uint64_t>(a, n), Modulus(q));
  });
}

int ref_reference_ntt(uint64_t n, uint64_t q, uint64_t psi, int dir, const uint64_t* a,
                      uint64_t* out) {
  return guarded([&] {
    auto v = reference_ntt(std::span<const uint64_t>(a, n), Modulus(q), psi,
                           dir == 0 ? NttDirection::forward : NttDirection::inverse);
    std::memcpy(out, v.data(), n * 8);
  });
}

int ref_naive_negacyclic(uint64_t n, uint64_t q, const uint64_t* f, const uint64_t* g,
                         uint64_t* out) {
  return guarded([&] {
    auto v = naive_negacyclic(std::span<const uint64_t>(f, n), std::span<const uint64_t>(g, n), q);
    std::memcpy(out, v.data(), n * 8);
  });
}

int ref_is_prime(uint64_t n) { return is_prime(n) ? 1 : 0; }

// harvey_forward_butterfly / harvey_inverse_butterfly (ntt.hpp:137-166) on
// element pairs, twiddle w with precompute_factor<bs>(w) (modarith.hpp:176-183)
int ref_butterflies(int fwd, uint64_t q, int bs, uint64_t w, const uint64_t* x0, const uint64_t* x1,
                    uint64_t n, uint64_t* y0, uint64_t* y1) {
  return guarded([&] {
    const Modulus m(q);
    for (uint64_t i = 0; i < n; ++i) {
      std::pair<uint64_t, uint64_t> r;
      if (bs == 52) {
        const MultiplyFactor f = precompute_factor<52>(w, m);
        r = fwd ? harvey_forward_butterfly<52>(x0[i], x1[i], f, m) : harvey_inverse_butterfly<52>(x0[i], x1[i], f, m);
      } else {
        const MultiplyFactor f = precompute_factor<64>(w, m);
        r = fwd ? harvey_forward_butterfly<64>(x0[i], x1[i], f, m) : harvey_inverse_butterfly<64>(x0[i], x1[i], f, m);
      }
      y0[i] = r.first;
      y1[i] = r.second;
    }
  });
}

}  // extern "C"
