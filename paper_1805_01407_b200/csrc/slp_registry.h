// Generator parameter table shared by the host library and the device kernels.
//
// Restates the reference registry (/root/reference/pkg/src/slprng/generators.py:71-110):
// the 18 sixty-four-bit and 7 thirty-two-bit named generators, then the two
// analysis baselines.  Word indices are in the flat (pointer-free) view of
// engines.py:14-18; `++` adds back the FIRST index (scramblers.py:34-38).
//
// X(id, name, family, k, w, a, b, c, scrambler, word_i, word_j, S, R, T)
//   family:    SLP_FAM_XOROSHIRO / SLP_FAM_XOSHIRO / SLP_FAM_XORSHIFT
//   scrambler: SLP_SC_NONE / PLUS / STAR / PLUSPLUS / STARSTAR
//   word_j = -1 when unused; c = 0 when the family has no third parameter.
#pragma once

#define SLP_FAM_XOROSHIRO 0
#define SLP_FAM_XOSHIRO 1
#define SLP_FAM_XORSHIFT 2

#define SLP_SC_NONE 0
#define SLP_SC_PLUS 1
#define SLP_SC_STAR 2
#define SLP_SC_PLUSPLUS 3
#define SLP_SC_STARSTAR 4

#define SLP_STAR64 0x9E3779B97F4A7C13ull
#define SLP_STAR32 0x9E3779BBull

// clang-format off
#define SLP_REGISTRY(X) \
  X( 0, xoroshiro128,          SLP_FAM_XOROSHIRO,  2, 64, 24, 16, 37, SLP_SC_NONE,     0, -1, 0ull,        0, 0ull) \
  X( 1, xoroshiro128plus,      SLP_FAM_XOROSHIRO,  2, 64, 24, 16, 37, SLP_SC_PLUS,     0,  1, 0ull,        0, 0ull) \
  X( 2, xoroshiro128star,      SLP_FAM_XOROSHIRO,  2, 64, 24, 16, 37, SLP_SC_STAR,     0, -1, SLP_STAR64,  0, 0ull) \
  X( 3, xoroshiro128plusplus,  SLP_FAM_XOROSHIRO,  2, 64, 49, 21, 28, SLP_SC_PLUSPLUS, 0,  1, 0ull,       17, 0ull) \
  X( 4, xoroshiro128starstar,  SLP_FAM_XOROSHIRO,  2, 64, 24, 16, 37, SLP_SC_STARSTAR, 0, -1, 5ull,        7, 9ull) \
  X( 5, xoshiro256,            SLP_FAM_XOSHIRO,    4, 64, 17, 45,  0, SLP_SC_NONE,     1, -1, 0ull,        0, 0ull) \
  X( 6, xoshiro256plus,        SLP_FAM_XOSHIRO,    4, 64, 17, 45,  0, SLP_SC_PLUS,     0,  3, 0ull,        0, 0ull) \
  X( 7, xoshiro256plusplus,    SLP_FAM_XOSHIRO,    4, 64, 17, 45,  0, SLP_SC_PLUSPLUS, 0,  3, 0ull,       23, 0ull) \
  X( 8, xoshiro256starstar,    SLP_FAM_XOSHIRO,    4, 64, 17, 45,  0, SLP_SC_STARSTAR, 1, -1, 5ull,        7, 9ull) \
  X( 9, xoshiro512,            SLP_FAM_XOSHIRO,    8, 64, 11, 21,  0, SLP_SC_NONE,     1, -1, 0ull,        0, 0ull) \
  X(10, xoshiro512plus,        SLP_FAM_XOSHIRO,    8, 64, 11, 21,  0, SLP_SC_PLUS,     0,  2, 0ull,        0, 0ull) \
  X(11, xoshiro512plusplus,    SLP_FAM_XOSHIRO,    8, 64, 11, 21,  0, SLP_SC_PLUSPLUS, 2,  0, 0ull,       17, 0ull) \
  X(12, xoshiro512starstar,    SLP_FAM_XOSHIRO,    8, 64, 11, 21,  0, SLP_SC_STARSTAR, 1, -1, 5ull,        7, 9ull) \
  X(13, xoroshiro1024,         SLP_FAM_XOROSHIRO, 16, 64, 25, 27, 36, SLP_SC_NONE,     0, -1, 0ull,        0, 0ull) \
  X(14, xoroshiro1024plus,     SLP_FAM_XOROSHIRO, 16, 64, 25, 27, 36, SLP_SC_PLUS,     0, 15, 0ull,        0, 0ull) \
  X(15, xoroshiro1024star,     SLP_FAM_XOROSHIRO, 16, 64, 25, 27, 36, SLP_SC_STAR,     0, -1, SLP_STAR64,  0, 0ull) \
  X(16, xoroshiro1024plusplus, SLP_FAM_XOROSHIRO, 16, 64, 25, 27, 36, SLP_SC_PLUSPLUS,15,  0, 0ull,       23, 0ull) \
  X(17, xoroshiro1024starstar, SLP_FAM_XOROSHIRO, 16, 64, 25, 27, 36, SLP_SC_STARSTAR, 0, -1, 5ull,        7, 9ull) \
  X(18, xoroshiro64,           SLP_FAM_XOROSHIRO,  2, 32, 26,  9, 13, SLP_SC_NONE,     0, -1, 0ull,        0, 0ull) \
  X(19, xoroshiro64star,       SLP_FAM_XOROSHIRO,  2, 32, 26,  9, 13, SLP_SC_STAR,     0, -1, SLP_STAR32,  0, 0ull) \
  X(20, xoroshiro64starstar,   SLP_FAM_XOROSHIRO,  2, 32, 26,  9, 13, SLP_SC_STARSTAR, 0, -1, SLP_STAR32,  5, 5ull) \
  X(21, xoshiro128,            SLP_FAM_XOSHIRO,    4, 32,  9, 11,  0, SLP_SC_NONE,     1, -1, 0ull,        0, 0ull) \
  X(22, xoshiro128plus,        SLP_FAM_XOSHIRO,    4, 32,  9, 11,  0, SLP_SC_PLUS,     0,  3, 0ull,        0, 0ull) \
  X(23, xoshiro128plusplus,    SLP_FAM_XOSHIRO,    4, 32,  9, 11,  0, SLP_SC_PLUSPLUS, 0,  3, 0ull,        7, 0ull) \
  X(24, xoshiro128starstar,    SLP_FAM_XOSHIRO,    4, 32,  9, 11,  0, SLP_SC_STARSTAR, 1, -1, 5ull,        7, 9ull) \
  X(25, xorshift128,           SLP_FAM_XORSHIFT,   2, 64, 23, 17, 26, SLP_SC_NONE,     0, -1, 0ull,        0, 0ull) \
  X(26, xorshift128plus,       SLP_FAM_XORSHIFT,   2, 64, 23, 17, 26, SLP_SC_PLUS,     0,  1, 0ull,        0, 0ull)
// clang-format on

#define SLP_NUM_GENERATORS 27
#define SLP_NUM_PRODUCTION 25

// Engine shapes (family, k, w) with run-time parameter kernel instances
// (GenR<>, slp_gen.cuh) for custom_spec engines (generators.py:127-135):
// the registry's engine shapes with any parameters, plus the 32-bit
// xorshift and 8-word xoshiro.  X(shape index, family, k, w)
// clang-format off
#define SLP_RT_SHAPES(X) \
  X(0, SLP_FAM_XOROSHIRO,  2, 64) \
  X(1, SLP_FAM_XOROSHIRO, 16, 64) \
  X(2, SLP_FAM_XOSHIRO,    4, 64) \
  X(3, SLP_FAM_XOSHIRO,    8, 64) \
  X(4, SLP_FAM_XORSHIFT,   2, 64) \
  X(5, SLP_FAM_XOROSHIRO,  2, 32) \
  X(6, SLP_FAM_XOSHIRO,    4, 32) \
  X(7, SLP_FAM_XOSHIRO,    8, 32) \
  X(8, SLP_FAM_XORSHIFT,   2, 32)
// clang-format on
#define SLP_NUM_RT_SHAPES 9
// ids of registered custom generators (slp_register_generator) start here
#define SLP_CUSTOM_ID0 1024
#define SLP_MAX_CUSTOM 4096
