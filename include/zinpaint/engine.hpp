// Forwarding header: the reference's include path zinpaint/engine.hpp
// (/root/reference/proj/include/zinpaint/engine.hpp) served by the B200 drop-in.
#pragma once
#include "../zinpaint_b200.hpp"
