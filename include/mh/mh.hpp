// mh/mh.hpp -- everything of the C++ mirror of the reference's header API
// (namespace mh), backed by libmhg.so on an sm_100 GPU.
//
//   geometry      mh/layout.hpp     Layout, encode, extract_i / extract_j
//   field         mh/field.hpp      Modulus, Fp, add, mul
//   containers    mh/matrix.hpp     Matrix (device store + host mirror), Grid,
//                                   from_row_major / to_row_major (device kernels)
//   views         mh/submatrix.hpp  Sub, Aligned, split_sub, quadrants, predicates
//   multiply      mh/multiply.hpp   Problem, Counters, mm_oblivious (+ Op::Sub / Op::Set),
//                                   mm_naive, mm_default, base_case_mm, compatible_parts,
//                                   mm_oblivious_async (explicit stream), synchronize
//   protocol      mh/bench.hpp      Config, Rng, gen_problem, run_trials, CSV writers
//   fixtures      mh/io.hpp         load_matrix / save_matrix text format
//   TU driver     mh/tu.hpp         schur_views, schur_update, SchurSweep (aliased Schur updates)
//
// Link with -lmhg (paper_1705_04807_b200/libmhg.so).
#pragma once

#define MH_B200_MIRROR 1

#include "mh/bench.hpp"
#include "mh/field.hpp"
#include "mh/io.hpp"
#include "mh/layout.hpp"
#include "mh/matrix.hpp"
#include "mh/multiply.hpp"
#include "mh/submatrix.hpp"
#include "mh/tu.hpp"
