// Stand-in for the reference header noma/format.hpp when the reference tree is
// absent: the whole API is declared in noma/detector.hpp.
#pragma once
#include "noma/detector.hpp"
