// Forwarding header: the reference's include path zinpaint/zcurve.hpp
// (/root/reference/proj/include/zinpaint/zcurve.hpp) served by the B200 drop-in.
#pragma once
#include "../zinpaint_b200.hpp"
