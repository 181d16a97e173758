// mh/mh.hpp -- umbrella header of the C++ mirror of the reference API
// (reference: proj/include/mh/mh.hpp), backed by libmhg.so on a B200.
#pragma once

#include "mh/bench.hpp"
#include "mh/field.hpp"
#include "mh/io.hpp"
#include "mh/layout.hpp"
#include "mh/matrix.hpp"
#include "mh/multiply.hpp"
#include "mh/submatrix.hpp"
