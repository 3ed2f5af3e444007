// Exercises the C++ facade (include/nttkit_b200.hpp) the way a caller of the
// reference's C++ API would. `--cpu`: only the argument-error behaviour (no
// device needed). Default: also transforms, element-wise and ring calls on the
// GPU, checked against known answers of the reference's tests.
#include <cstdio>
#include <cstring>
#include <optional>
#include <random>
#include <stdexcept>
#include <vector>

#include "../../include/nttkit_b200.hpp"

namespace nb = nttkit_b200;

static int failures = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

template <class F>
static bool throws_invalid(F&& f) {
  try {
    f();
  } catch (const std::invalid_argument&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu") == 0;
  // modarith.hpp:109-111 / test_modarith.cpp:31-42
  EXPECT(throws_invalid([] { nb::Modulus m(15); }));
  EXPECT(throws_invalid([] { nb::Modulus m(2); }));
  EXPECT(nb::Modulus(17).bits() == 5);
  // ntt.hpp:219-236 / test_ntt.cpp:57-70 (validated before any device work)
  EXPECT(throws_invalid([] { nb::NttTables t(4, nb::Modulus(13)); }));
  EXPECT(throws_invalid([] { nb::NttTables t(3, nb::Modulus(17)); }));
  EXPECT(throws_invalid([] { nb::NttTables t(4, nb::Modulus(17), std::nullopt, 48); }));
  EXPECT(throws_invalid([] { nb::NttTables t(4, nb::Modulus(17), uint64_t{3}); }));
  // modarith.hpp:176-183 / test_modarith.cpp:195
  EXPECT(nb::precompute_factor<64>(1, nb::Modulus(17)).precon == 1085102592571150095ull);
  EXPECT(throws_invalid([] { nb::precompute_factor<64>(17, nb::Modulus(17)); }));
  // ntt.hpp:37-58 / test_ntt.cpp: bit reversal and its permutation (host only)
  EXPECT(nb::bit_reverse(1, 3) == 4 && nb::bit_reverse(6, 3) == 3 && nb::bit_reverse(0, 0) == 0);
  EXPECT(throws_invalid([] { (void)nb::bit_reverse(8, 3); }));
  {
    std::vector<uint64_t> p{0, 1, 2, 3, 4, 5, 6, 7};
    nb::bit_reverse_permute(std::span<uint64_t>(p));
    EXPECT((p == std::vector<uint64_t>{0, 4, 2, 6, 1, 5, 3, 7}));
    nb::bit_reverse_permute(std::span<uint64_t>(p));
    EXPECT((p == std::vector<uint64_t>{0, 1, 2, 3, 4, 5, 6, 7}));
    std::vector<uint64_t> bad(6);
    EXPECT(throws_invalid([&] { nb::bit_reverse_permute(std::span<uint64_t>(bad)); }));
  }
  // test_ntt.cpp:37-43: minimal primitive roots
  EXPECT(nb::minimal_primitive_root(4, nb::Modulus(17)) == 4);
  EXPECT(nb::minimal_primitive_root(2, nb::Modulus(5)) == 4);
  EXPECT(nb::minimal_primitive_root(8, nb::Modulus(17)) == 2);  // NttTables(4, 17).root()
  EXPECT(nb::minimal_primitive_root(4, nb::Modulus(5)) == 2);   // NttTables(2, 5).root()
  EXPECT(throws_invalid([] { (void)nb::minimal_primitive_root(3, nb::Modulus(17)); }));
  if (cpu_only) {
    std::printf(failures ? "facade cpu checks FAILED\n" : "facade cpu checks ok\n");
    return failures ? 1 : 0;
  }
  // test_ntt.cpp:44-55 (TableLayout): accessors of NttTables(4, 17), psi = 2
  {
    const nb::Modulus m(17);
    const nb::NttTables t(4, m);
    EXPECT(t.log2_size() == 2 && t.size() == 4 && t.root() == 2 && t.bit_shift() == 52);  // 4q < 2^52
    EXPECT(t.inv_root() == 9);  // 2 * 9 = 18 == 1 (mod 17)
    uint64_t p = 1;
    for (uint64_t i = 0; i < 4; ++i) {
      EXPECT(t.root_powers_rev()[nb::bit_reverse(i, 2)] == p);
      const unsigned __int128 pre = (static_cast<unsigned __int128>(p) << 52) / 17;
      EXPECT(t.root_precons_rev()[nb::bit_reverse(i, 2)] == static_cast<uint64_t>(pre));
      p = p * 2 % 17;
    }
    uint64_t pi = 1;
    for (uint64_t i = 0; i < 4; ++i) {
      EXPECT(t.inv_root_powers_rev()[nb::bit_reverse(i, 2)] == pi);
      pi = pi * 9 % 17;
    }
    EXPECT(t.inv_root_precons_rev().size() == 4);
    EXPECT(t.inv_size().operand * 4 % 17 == 1);
    EXPECT(t.inv_size() == nb::precompute_factor<52>(t.inv_size().operand, m));
  }
  // test_ntt.cpp:94-114: n=2, q=5
  nb::NttTables t2(2, nb::Modulus(5));
  EXPECT(t2.root() == 2);
  std::vector<uint64_t> a{1, 1}, out(2);
  t2.forward(out, a, 1, 1);
  EXPECT(out[0] == 3 && out[1] == 4);
  t2.inverse(out, out, 1, 1);
  EXPECT(out[0] == 1 && out[1] == 1);
  EXPECT(throws_invalid([&] { t2.forward(out, a, 3, 1); }));
  // round trip at cfg1 size through the HEXL names
  const uint64_t q = 1125899906826241ull;
  nb::hexl::NTT ntt(4096, q);
  std::mt19937_64 eng(1 ^ 20260809);
  std::vector<uint64_t> x(4096), y(4096), z(4096);
  for (auto& v : x) v = eng() % q;
  ntt.ComputeForward(y.data(), x.data(), 1, 1);
  ntt.ComputeInverse(z.data(), y.data(), 1, 1);
  EXPECT(z == x);
  // test_eltwise.cpp:180-186: 2*3+4 mod 17 = 10
  uint64_t r = 0, two = 2, four = 4;
  nb::hexl::EltwiseFMAMod(&r, &two, 3, &four, 1, 17, 1);
  EXPECT(r == 10);
  // (q-1)^2 == 1
  std::vector<uint64_t> top(64, q - 1), one(64);
  nb::hexl::EltwiseMultMod(one.data(), top.data(), top.data(), 64, q, 1);
  for (auto v : one) EXPECT(v == 1);
  // test_ring.cpp:41-54: X * X^(n-1) = -1 mod (X^8 + 1, 97)
  nb::NttTables t8(8, nb::Modulus(97));
  std::vector<uint64_t> xa(8, 0), xb(8, 0), xc(8);
  xa[1] = 1;
  xb[7] = 1;
  nb::poly_mult_mod(xc, xa, xb, t8);
  EXPECT(xc[0] == 96);
  for (int i = 1; i < 8; ++i) EXPECT(xc[i] == 0);
  // CoeffVec overloads (ntt.hpp:308-320, eltwise.hpp:273-303, ring.hpp:45-51)
  {
    nb::CoeffVec cx(x, 1);
    const nb::CoeffVec fx = ntt.GetDegree() == 4096 ? nb::NttTables(4096, nb::Modulus(q)).forward(cx, 1, 4)
                                                    : nb::CoeffVec();
    EXPECT(fx.bound_factor == 4 && fx.within_bound(nb::Modulus(q)));
    const nb::CoeffVec back = nb::NttTables(4096, nb::Modulus(q)).inverse(
        nb::NttTables(4096, nb::Modulus(q)).forward(cx, 1, 1), 1, 1);
    EXPECT(back.data == x);
    const nb::Modulus m97(97);
    nb::CoeffVec a5(std::vector<uint64_t>{1, 96, 50, 0}, 1), b5(std::vector<uint64_t>{96, 96, 50, 0}, 1);
    EXPECT((nb::eltwise_add_mod(a5, b5, m97).data == std::vector<uint64_t>{0, 95, 3, 0}));
    EXPECT((nb::eltwise_neg_mod(a5, m97).data == std::vector<uint64_t>{96, 1, 47, 0}));
    EXPECT((nb::eltwise_mult_mod(a5, b5, m97, 1).data == std::vector<uint64_t>{96, 1, 75, 0}));
    EXPECT(throws_invalid([&] { nb::eltwise_mult_mod(nb::CoeffVec(a5.data, 2), b5, m97, 1); }));
    nb::CoeffVec p1(std::vector<uint64_t>(8, 0), 1), p2(std::vector<uint64_t>(8, 0), 1);
    p1.data[1] = 1;
    p2.data[7] = 1;
    EXPECT(nb::poly_mult_mod(p1, p2, t8).data[0] == 96);
  }
  // test_ntt.cpp:264-275: the public butterflies
  {
    const nb::Modulus m17(17);
    const auto f5 = nb::precompute_factor<64>(5, m17);
    const auto [y0, y1] = nb::harvey_forward_butterfly<64>(0, 0, f5, m17);
    EXPECT(y0 == 0 && y1 == 34);
    const auto f3 = nb::precompute_factor<52>(3, m17);
    const auto [z0, z1] = nb::harvey_inverse_butterfly<52>(7, 7, f3, m17);
    EXPECT(z0 % 17 == 14 && z1 % 17 == 0);
  }
  std::printf(failures ? "facade gpu checks FAILED\n" : "facade gpu checks ok\n");
  return failures ? 1 : 0;
}
