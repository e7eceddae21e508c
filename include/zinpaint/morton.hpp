// Forwarding header: the reference's include path zinpaint/morton.hpp
// (/root/reference/proj/include/zinpaint/morton.hpp) served by the B200 drop-in.
#pragma once
#include "../zinpaint_b200.hpp"
