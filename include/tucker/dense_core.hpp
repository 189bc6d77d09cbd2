#pragma once
// B200 drop-in: the dense_core.hpp names live in tucker_b200.hpp
#include "tucker/tucker_b200.hpp"
