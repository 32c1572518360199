// bitkv/serialize.hpp -> the B200 drop-in (include/bitkv_b200.hpp)
#pragma once
#include "bitkv_b200.hpp"
