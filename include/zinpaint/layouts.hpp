// Forwarding header: the reference's include path zinpaint/layouts.hpp
// (/root/reference/proj/include/zinpaint/layouts.hpp) served by the B200 drop-in.
#pragma once
#include "../zinpaint_b200.hpp"
