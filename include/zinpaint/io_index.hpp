// Forwarding header: the reference's include path zinpaint/io_index.hpp
// (/root/reference/proj/include/zinpaint/io_index.hpp) served by the B200 drop-in.
#pragma once
#include "../zinpaint_b200.hpp"
