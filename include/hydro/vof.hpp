// hydro/vof.hpp — forwards to the B200 drop-in (see hydro/b200.hpp).
#pragma once
#include "hydro/b200.hpp"
