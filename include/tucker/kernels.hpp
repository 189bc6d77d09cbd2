#pragma once
// B200 drop-in: the kernels.hpp names live in tucker_b200.hpp
#include "tucker/tucker_b200.hpp"
