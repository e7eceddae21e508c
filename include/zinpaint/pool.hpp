// Forwarding header: the reference's include path zinpaint/pool.hpp
// (/root/reference/proj/include/zinpaint/pool.hpp) served by the B200 drop-in.
#pragma once
#include "../zinpaint_b200.hpp"
