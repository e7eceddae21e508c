// Forwarding header: the reference's include path zinpaint/types.hpp
// (/root/reference/proj/include/zinpaint/types.hpp) served by the B200 drop-in.
#pragma once
#include "../zinpaint_b200.hpp"
