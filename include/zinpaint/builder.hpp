// Forwarding header: the reference's include path zinpaint/builder.hpp
// (/root/reference/proj/include/zinpaint/builder.hpp) served by the B200 drop-in.
#pragma once
#include "../zinpaint_b200.hpp"
