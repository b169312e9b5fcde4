// Drop-in path shim: the reference header gopt/precision.hpp maps onto the B200 facade.
#pragma once
#include "../gopt.hpp"
