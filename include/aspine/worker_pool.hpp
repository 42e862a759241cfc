// Reference include path /root/reference/proj/include/aspine/worker_pool.hpp: the
// yasmin-b200 C++ facade provides it (include/yasmin/aspine.hpp).
#pragma once
#include "../yasmin/aspine.hpp"
