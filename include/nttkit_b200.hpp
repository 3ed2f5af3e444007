// nttkit_b200.hpp — header-only C++ facade over the C-ABI (nttkit_b200.h),
// mirroring the reference's C++ API (/root/reference/proj/include/nttkit/) so
// a caller of the reference can switch by changing the namespace:
//
//   reference (nttkit::)                        this facade (nttkit_b200::)
//   Modulus(q)                modarith.hpp:106  Modulus(q)
//   bit_reverse(i, log2n)     ntt.hpp:37-46     bit_reverse (host)
//   bit_reverse_permute(v)    ntt.hpp:49-58     bit_reverse_permute (host)
//   minimal_primitive_root    ntt.hpp:172-197   minimal_primitive_root (host)
//   NttTables(n, m[, root])   ntt.hpp:210-217   NttTables(n, m[, root][, bit_shift])
//   NttTables accessors       ntt.hpp:249-261   size, log2_size, modulus, root, inv_root,
//                                               bit_shift, inv_size, root_powers_rev,
//                                               root_precons_rev, inv_root_powers_rev,
//                                               inv_root_precons_rev (host copies)
//   NttTables::forward        ntt.hpp:268-285   NttTables::forward (host spans)
//   NttTables::inverse        ntt.hpp:289-306   NttTables::inverse (host spans)
//   eltwise_mult_mod          eltwise.hpp:180   eltwise_mult_mod
//   eltwise_mult_mod_int      eltwise.hpp:137   eltwise_mult_mod_int
//   precompute_factor<B>      modarith.hpp:176  precompute_factor
//   harvey_*_butterfly<B>     ntt.hpp:137,154   harvey_forward/inverse_butterfly
//   eltwise_mult_mod_float    eltwise.hpp:158   eltwise_mult_mod_float
//   eltwise_fma_mod           eltwise.hpp:263   eltwise_fma_mod (std::optional addend)
//   poly_mult_mod             ring.hpp:28-43    poly_mult_mod
//   HEXL: hexl::NTT{ComputeForward, ComputeInverse},
//                            hexl::EltwiseMultMod, hexl::EltwiseFMAMod
//
// Host-span calls copy to the GPU, run the sm_100a kernels and copy back before
// returning (the reference's calls are blocking). Argument errors throw
// std::invalid_argument with the reference's message; CUDA failures throw
// std::runtime_error. RnsNtt exposes the batched device-pointer entry points.
#ifndef NTTKIT_B200_HPP
#define NTTKIT_B200_HPP

#include <cstdint>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "nttkit_b200.h"

namespace nttkit_b200 {

inline void check(int rc) {
  if (rc == NK_OK) return;
  const std::string msg = nk_last_error();
  if (rc == NK_ERR_CUDA) throw std::runtime_error(msg);
  throw std::invalid_argument(msg);
}

class Modulus {
 public:
  explicit Modulus(uint64_t q) : q_(q) { check(nk_modulus(q, &bits_, &barrett_)); }
  uint64_t value() const noexcept { return q_; }
  unsigned bits() const noexcept { return bits_; }
  unsigned barrett_shift() const noexcept { return 63 + bits_; }
  uint64_t barrett_factor() const noexcept { return barrett_; }
  friend bool operator==(const Modulus& a, const Modulus& b) { return a.q_ == b.q_; }

 private:
  uint64_t q_;
  uint32_t bits_ = 0;
  uint64_t barrett_ = 0;
};

/// Residue vector with its declared range bound (ntt.hpp:60-80): every element
/// is promised to be below bound_factor * q (bookkeeping for the lazy
/// contracts; checked by within_bound).
struct CoeffVec {
  std::vector<uint64_t> data;
  uint64_t bound_factor = 1;
  CoeffVec() = default;
  explicit CoeffVec(std::vector<uint64_t> d, uint64_t factor = 1) : data(std::move(d)), bound_factor(factor) {}
  uint64_t size() const noexcept { return data.size(); }
  bool within_bound(const Modulus& m) const {
    const unsigned __int128 bound = static_cast<unsigned __int128>(bound_factor) * m.value();
    for (uint64_t x : data)
      if (x >= bound) return false;
    return true;
  }
};

/// precompute_factor<BitShift> (modarith.hpp:168-183)
struct MultiplyFactor {
  uint64_t operand;
  uint64_t precon;
  friend bool operator==(const MultiplyFactor&, const MultiplyFactor&) = default;
};

/// Reverse the low log2n bits of i (ntt.hpp:37-46). The reference checks the
/// contract in checked builds; here a violation throws std::invalid_argument.
constexpr uint64_t bit_reverse(uint64_t i, unsigned log2n) {
  if (!(log2n < 64 && (log2n == 0 ? i == 0 : i >> log2n == 0)))
    throw std::invalid_argument("bit_reverse: index must have log2n bits");
  uint64_t r = 0;
  for (unsigned b = 0; b < log2n; ++b) {
    r = (r << 1) | (i & 1);
    i >>= 1;
  }
  return r;
}

/// In-place bit-reversal permutation of a power-of-two-length span (an
/// involution; ntt.hpp:49-58).
template <typename T>
void bit_reverse_permute(std::span<T> v) {
  const uint64_t n = v.size();
  if (n == 0 || (n & (n - 1)) != 0)
    throw std::invalid_argument("bit_reverse_permute: length must be a power of two");
  unsigned log2n = 0;
  while ((uint64_t{1} << log2n) < n) ++log2n;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t j = bit_reverse(i, log2n);
    if (i < j) std::swap(v[i], v[j]);
  }
}

/// Smallest primitive `order`'th root of unity mod q (ntt.hpp:172-197), the
/// root NttTables uses when none is supplied.
inline uint64_t minimal_primitive_root(uint64_t order, const Modulus& m) {
  uint64_t r = 0;
  check(nk_minimal_primitive_root(order, m.value(), &r));
  return r;
}

// Tables of many RNS limbs on one device; batched data is [npolys][nlimbs][n].
class RnsNtt {
 public:
  RnsNtt(uint64_t n, std::span<const uint64_t> moduli, int device = 0, int bit_shift = 0,
         std::optional<std::span<const uint64_t>> roots = std::nullopt) {
    nk_plan* p = nullptr;
    check(nk_plan_create(&p, device, n, moduli.data(), roots ? roots->data() : nullptr,
                         static_cast<uint32_t>(moduli.size()), bit_shift));
    plan_.reset(p);
    n_ = n;
    nlimbs_ = static_cast<uint32_t>(moduli.size());
  }
  uint64_t size() const noexcept { return n_; }
  uint32_t limbs() const noexcept { return nlimbs_; }
  const nk_plan* plan() const noexcept { return plan_.get(); }

  // device pointers, asynchronous on `stream` (cudaStream_t)
  void forward_device(uint64_t* d_result, const uint64_t* d_operand, uint32_t npolys,
                      uint64_t in, uint64_t out, void* stream = nullptr) const {
    check(nk_ntt_forward(plan_.get(), d_result, d_operand, 0, nlimbs_, npolys, in, out, stream));
  }
  void inverse_device(uint64_t* d_result, const uint64_t* d_operand, uint32_t npolys,
                      uint64_t in, uint64_t out, void* stream = nullptr) const {
    check(nk_ntt_inverse(plan_.get(), d_result, d_operand, 0, nlimbs_, npolys, in, out, stream));
  }
  void poly_mult_device(uint64_t* d_result, const uint64_t* d_f, const uint64_t* d_g,
                        uint32_t npolys, void* stream = nullptr) const {
    check(nk_poly_mult_mod(plan_.get(), d_result, d_f, d_g, 0, nlimbs_, npolys, stream));
  }

  // host buffers, blocking
  void forward(std::span<uint64_t> result, std::span<const uint64_t> operand, uint64_t in,
               uint64_t out) const {
    host_call(true, result, operand, in, out);
  }
  void inverse(std::span<uint64_t> result, std::span<const uint64_t> operand, uint64_t in,
               uint64_t out) const {
    host_call(false, result, operand, in, out);
  }

 protected:
  void host_call(bool fwd, std::span<uint64_t> result, std::span<const uint64_t> operand,
                 uint64_t in, uint64_t out) const {
    const uint64_t row = n_ * nlimbs_;
    if (operand.size() != result.size() || row == 0 || operand.size() % row != 0)
      throw std::invalid_argument("transform: buffer length must equal n");
    const uint32_t npolys = static_cast<uint32_t>(operand.size() / row);
    auto fn = fwd ? nk_ntt_forward_host : nk_ntt_inverse_host;
    check(fn(plan_.get(), result.data(), operand.data(), operand.size(), 0, nlimbs_, npolys, in,
             out, nullptr));
  }

  struct Deleter {
    void operator()(nk_plan* p) const { nk_plan_destroy(p); }
  };
  std::unique_ptr<nk_plan, Deleter> plan_;
  uint64_t n_ = 0;
  uint32_t nlimbs_ = 0;
};

// NttTables(n, Modulus[, root][, bit_shift]) — one limb, reference semantics.
class NttTables : public RnsNtt {
 public:
  NttTables(uint64_t n, const Modulus& m) : RnsNtt(n, one(m)), m_(m) { build_host(); }
  NttTables(uint64_t n, const Modulus& m, uint64_t root)
      : RnsNtt(n, one(m), 0, 0, std::span<const uint64_t>(&root_holder(root), 1)), m_(m) {
    build_host();
  }
  NttTables(uint64_t n, const Modulus& m, std::optional<uint64_t> root, int bit_shift)
      : RnsNtt(n, one(m), 0, bit_shift,
               root ? std::optional<std::span<const uint64_t>>(
                          std::span<const uint64_t>(&root_holder(*root), 1))
                    : std::nullopt),
        m_(m) {
    // the reference validates the width before it looks at a root (ntt.hpp:226-231);
    // nk_plan_create applies the same order.
    build_host();
  }
  const Modulus& modulus() const noexcept { return m_; }
  unsigned log2_size() const noexcept {
    unsigned l = 0;
    while ((uint64_t{1} << l) < size()) ++l;
    return l;
  }
  uint64_t root() const { return host().psi; }
  /// psi^-1: the inverse table holds psi^-i at bit_reverse(i), so psi^-1 sits at n/2
  uint64_t inv_root() const { return host().wi[size() / 2]; }
  int bit_shift() const { return host().bs; }
  /// n^-1 mod q with its precon for the table width (ntt.hpp:259)
  MultiplyFactor inv_size() const { return {host().ninv, host().ninvp}; }
  /// psi^i at index bit_reverse(i), with the matching precon array (ntt.hpp:256-261);
  /// copies of the tables the device plan was built from, bit for bit the
  /// reference's build_tables (ntt.hpp:343-361)
  std::span<const uint64_t> root_powers_rev() const { return host().w; }
  std::span<const uint64_t> root_precons_rev() const { return host().wp; }
  std::span<const uint64_t> inv_root_powers_rev() const { return host().wi; }
  std::span<const uint64_t> inv_root_precons_rev() const { return host().wip; }
  void forward(std::span<uint64_t> result, std::span<const uint64_t> operand, uint64_t in,
               uint64_t out) const {
    if (result.size() != size() || operand.size() != size())
      throw std::invalid_argument("transform: buffer length must equal n");
    host_call(true, result, operand, in, out);
  }
  void inverse(std::span<uint64_t> result, std::span<const uint64_t> operand, uint64_t in,
               uint64_t out) const {
    if (result.size() != size() || operand.size() != size())
      throw std::invalid_argument("transform: buffer length must equal n");
    host_call(false, result, operand, in, out);
  }
  // CoeffVec overloads (ntt.hpp:308-320): the result carries output_mod_factor
  CoeffVec forward(const CoeffVec& in, uint64_t input_mod_factor, uint64_t output_mod_factor) const {
    if (in.bound_factor > input_mod_factor)
      throw std::invalid_argument("forward: CoeffVec bound exceeds input_mod_factor");
    CoeffVec out(std::vector<uint64_t>(in.data.size()), output_mod_factor);
    forward(out.data, in.data, input_mod_factor, output_mod_factor);
    return out;
  }
  CoeffVec inverse(const CoeffVec& in, uint64_t input_mod_factor, uint64_t output_mod_factor) const {
    if (in.bound_factor > input_mod_factor)
      throw std::invalid_argument("inverse: CoeffVec bound exceeds input_mod_factor");
    CoeffVec out(std::vector<uint64_t>(in.data.size()), output_mod_factor);
    inverse(out.data, in.data, input_mod_factor, output_mod_factor);
    return out;
  }

 private:
  static std::span<const uint64_t> one(const Modulus& m) {
    thread_local uint64_t q;
    q = m.value();
    return std::span<const uint64_t>(&q, 1);
  }
  static uint64_t& root_holder(uint64_t r) {
    thread_local uint64_t v;
    v = r;
    return v;
  }
  struct HostTables {
    uint64_t psi = 0, ninv = 0, ninvp = 0;
    int bs = 0;
    std::vector<uint64_t> w, wp, wi, wip;
  };
  // built once at construction from the plan's own (n, q, root, width), host
  // side only; immutable afterwards (concurrent const calls are safe, ntt.hpp:203-205)
  const HostTables& host() const { return *host_; }
  void build_host() {
    {
      auto h = std::make_shared<HostTables>();
      const uint64_t n = size();
      h->w.resize(n);
      h->wp.resize(n);
      h->wi.resize(n);
      h->wip.resize(n);
      uint64_t psi = 0;
      int bs = 0;
      check(nk_plan_info(plan(), 0, nullptr, nullptr, &psi, &bs, nullptr));
      check(nk_tables_host(n, m_.value(), &psi, bs, &h->psi, h->w.data(), h->wp.data(), h->wi.data(),
                           h->wip.data(), &h->ninv, &h->ninvp, &h->bs));
      host_ = std::move(h);
    }
  }
  Modulus m_;
  std::shared_ptr<const HostTables> host_;
};

inline void eltwise_mult_mod(std::span<uint64_t> result, std::span<const uint64_t> a,
                             std::span<const uint64_t> b, const Modulus& m,
                             uint64_t input_mod_factor) {
  if (result.size() != a.size() || a.size() != b.size())
    throw std::invalid_argument("eltwise: operand lengths must match");
  check(nk_eltwise_mult_mod_host(result.data(), a.data(), b.data(), a.size(), m.value(),
                                 input_mod_factor, 0, nullptr));
}


template <int BitShift>
inline MultiplyFactor precompute_factor(uint64_t w, const Modulus& m) {
  static_assert(BitShift == 52 || BitShift == 64, "accumulator width is 52 or 64");
  uint64_t p = 0;
  check(nk_precompute_factor(w, m.value(), BitShift, &p));
  return {w, p};
}

/// harvey_forward_butterfly / harvey_inverse_butterfly (ntt.hpp:137-166), run
/// on the GPU in the reference's integer arithmetic (a kernel launch per
/// call: the scalar API exists for parity; batched work goes through the
/// transforms).
template <int BitShift>
inline std::pair<uint64_t, uint64_t> harvey_forward_butterfly(uint64_t x0, uint64_t x1, const MultiplyFactor& w,
                                                              const Modulus& m) {
  uint64_t y0 = 0, y1 = 0;
  check(nk_harvey_butterflies(1, m.value(), BitShift, w.operand, w.precon, &x0, &x1, 1, &y0, &y1, 0));
  return {y0, y1};
}
template <int BitShift>
inline std::pair<uint64_t, uint64_t> harvey_inverse_butterfly(uint64_t x0, uint64_t x1, const MultiplyFactor& w,
                                                              const Modulus& m) {
  uint64_t y0 = 0, y1 = 0;
  check(nk_harvey_butterflies(0, m.value(), BitShift, w.operand, w.precon, &x0, &x1, 1, &y0, &y1, 0));
  return {y0, y1};
}

inline void eltwise_mult_mod_int(std::span<uint64_t> result, std::span<const uint64_t> a,
                                 std::span<const uint64_t> b, const Modulus& m,
                                 uint64_t input_mod_factor) {
  if (result.size() != a.size() || a.size() != b.size())
    throw std::invalid_argument("eltwise: operand lengths must match");
  check(nk_eltwise_mult_mod_int_host(result.data(), a.data(), b.data(), a.size(), m.value(),
                                     input_mod_factor, 0, nullptr));
}

inline void eltwise_mult_mod_float(std::span<uint64_t> result, std::span<const uint64_t> a,
                                   std::span<const uint64_t> b, const Modulus& m,
                                   uint64_t input_mod_factor) {
  if (result.size() != a.size() || a.size() != b.size())
    throw std::invalid_argument("eltwise: operand lengths must match");
  check(nk_eltwise_mult_mod_float_host(result.data(), a.data(), b.data(), a.size(), m.value(),
                                       input_mod_factor, 0, nullptr));
}

inline void eltwise_fma_mod(std::span<uint64_t> result, std::span<const uint64_t> a, uint64_t y,
                            std::optional<std::span<const uint64_t>> z, const Modulus& m,
                            uint64_t input_mod_factor) {
  if (result.size() != a.size() || (z && z->size() != a.size()))
    throw std::invalid_argument("eltwise: operand lengths must match");
  check(nk_eltwise_fma_mod_host(result.data(), a.data(), y, z ? z->data() : nullptr, a.size(),
                                m.value(), input_mod_factor, 0, 0, nullptr));
}

inline void poly_mult_mod(std::span<uint64_t> result, std::span<const uint64_t> f,
                          std::span<const uint64_t> g, const NttTables& tables) {
  if (result.size() != tables.size() || f.size() != tables.size() || g.size() != tables.size())
    throw std::invalid_argument("poly_mult_mod: operand lengths must equal n");
  check(nk_poly_mult_mod_host(tables.plan(), result.data(), f.data(), g.data(), f.size(), 0, 1, 1,
                              nullptr));
}

inline void eltwise_add_mod(std::span<uint64_t> result, std::span<const uint64_t> a,
                            std::span<const uint64_t> b, const Modulus& m) {
  if (result.size() != a.size() || a.size() != b.size())
    throw std::invalid_argument("eltwise: operand lengths must match");
  check(nk_eltwise_add_mod_host(result.data(), a.data(), b.data(), a.size(), m.value(), 0, nullptr));
}

inline void eltwise_neg_mod(std::span<uint64_t> result, std::span<const uint64_t> a, const Modulus& m) {
  if (result.size() != a.size()) throw std::invalid_argument("eltwise: operand lengths must match");
  check(nk_eltwise_neg_mod_host(result.data(), a.data(), a.size(), m.value(), 0, nullptr));
}

// CoeffVec conveniences (eltwise.hpp:273-303, ring.hpp:45-51); results are fully reduced
inline CoeffVec eltwise_add_mod(const CoeffVec& a, const CoeffVec& b, const Modulus& m) {
  CoeffVec out(std::vector<uint64_t>(a.size()), 1);
  eltwise_add_mod(out.data, a.data, b.data, m);
  return out;
}
inline CoeffVec eltwise_neg_mod(const CoeffVec& a, const Modulus& m) {
  CoeffVec out(std::vector<uint64_t>(a.size()), 1);
  eltwise_neg_mod(out.data, a.data, m);
  return out;
}
inline CoeffVec eltwise_mult_mod(const CoeffVec& a, const CoeffVec& b, const Modulus& m,
                                 uint64_t input_mod_factor) {
  if (a.bound_factor > input_mod_factor || b.bound_factor > input_mod_factor)
    throw std::invalid_argument("eltwise_mult_mod: CoeffVec bound exceeds input_mod_factor");
  CoeffVec out(std::vector<uint64_t>(a.size()), 1);
  eltwise_mult_mod(out.data, a.data, b.data, m, input_mod_factor);
  return out;
}
inline CoeffVec eltwise_fma_mod(const CoeffVec& a, uint64_t y, const CoeffVec* z, const Modulus& m,
                                uint64_t input_mod_factor) {
  CoeffVec out(std::vector<uint64_t>(a.size()), 1);
  std::optional<std::span<const uint64_t>> zs;
  if (z != nullptr) zs = std::span<const uint64_t>(z->data);
  eltwise_fma_mod(out.data, a.data, y, zs, m, input_mod_factor);
  return out;
}
inline CoeffVec poly_mult_mod(const CoeffVec& f, const CoeffVec& g, const NttTables& tables) {
  if (f.bound_factor != 1 || g.bound_factor != 1)
    throw std::invalid_argument("poly_mult_mod: operands must be fully reduced");
  CoeffVec out(std::vector<uint64_t>(f.size()), 1);
  poly_mult_mod(out.data, f.data, g.data, tables);
  return out;
}

// ---- Intel HEXL names ----
namespace hexl {

class NTT {
 public:
  NTT(uint64_t degree, uint64_t q) : t_(degree, Modulus(q)) {}
  NTT(uint64_t degree, uint64_t q, uint64_t root_of_unity) : t_(degree, Modulus(q), root_of_unity) {}
  void ComputeForward(uint64_t* result, const uint64_t* operand, uint64_t input_mod_factor,
                      uint64_t output_mod_factor) const {
    t_.forward(std::span<uint64_t>(result, t_.size()), std::span<const uint64_t>(operand, t_.size()),
               input_mod_factor, output_mod_factor);
  }
  void ComputeInverse(uint64_t* result, const uint64_t* operand, uint64_t input_mod_factor,
                      uint64_t output_mod_factor) const {
    t_.inverse(std::span<uint64_t>(result, t_.size()), std::span<const uint64_t>(operand, t_.size()),
               input_mod_factor, output_mod_factor);
  }
  uint64_t GetDegree() const { return t_.size(); }
  uint64_t GetModulus() const { return t_.modulus().value(); }

 private:
  NttTables t_;
};

inline void EltwiseMultMod(uint64_t* result, const uint64_t* operand1, const uint64_t* operand2,
                           uint64_t n, uint64_t modulus, uint64_t input_mod_factor) {
  eltwise_mult_mod(std::span<uint64_t>(result, n), std::span<const uint64_t>(operand1, n),
                   std::span<const uint64_t>(operand2, n), Modulus(modulus), input_mod_factor);
}

// arg3 == nullptr: vector-scalar multiply
inline void EltwiseFMAMod(uint64_t* result, const uint64_t* arg1, uint64_t arg2,
                          const uint64_t* arg3, uint64_t n, uint64_t modulus,
                          uint64_t input_mod_factor) {
  std::optional<std::span<const uint64_t>> z;
  if (arg3) z = std::span<const uint64_t>(arg3, n);
  eltwise_fma_mod(std::span<uint64_t>(result, n), std::span<const uint64_t>(arg1, n), arg2, z,
                  Modulus(modulus), input_mod_factor);
}

}  // namespace hexl
}  // namespace nttkit_b200

#endif
