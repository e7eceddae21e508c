// Forwarding header: the reference's include path zinpaint/image.hpp
// (/root/reference/proj/include/zinpaint/image.hpp) served by the B200 drop-in.
#pragma once
#include "../zinpaint_b200.hpp"
