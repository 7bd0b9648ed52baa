# Build of the fvlog sm_100a runtime (in-tree, so the .so travels with the repo
# snapshot to the GPU box). `python -c "import __graft_entry__ as g; g.build()"`
# drives this file.
NVCC := /usr/local/cuda/bin/nvcc
HOSTCXX := /usr/bin/g++
PKG := paper_2501_13051_b200
SRC := $(PKG)/csrc
OBJ := build/obj
ARCH := -gencode arch=compute_100a,code=sm_100a

NVFLAGS := -std=c++17 -O3 $(ARCH) -lineinfo -ccbin $(HOSTCXX) -Xcompiler -fPIC -Xcompiler -g \
           -Iinclude -I$(SRC) --expt-relaxed-constexpr -Xptxas -warn-spills
CXXFLAGS := -std=c++17 -O2 -g -fPIC -Wall -Wextra -Wno-unused-parameter -Iinclude -I$(SRC) \
            -I/usr/local/cuda/include

CU_SRCS := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
HDRS := $(wildcard $(SRC)/*.h $(SRC)/*.cuh) include/fvlog.h
OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CU_SRCS)) $(patsubst $(SRC)/%.cpp,$(OBJ)/%.o,$(CPP_SRCS))

all: $(PKG)/libfvlog.so $(PKG)/fvlog tools/fvlog_membench tools/fvlog_sortbench tools/fvlog_scanbench

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(HOSTCXX) $(CXXFLAGS) -c $< -o $@

$(PKG)/libfvlog.so: $(OBJS)
	$(NVCC) $(ARCH) -ccbin $(HOSTCXX) -shared -o $@ $(OBJS) -cudart static -lpthread

$(PKG)/fvlog: tools/fvlog_main.cpp $(PKG)/libfvlog.so
	$(HOSTCXX) -std=c++17 -O2 -Iinclude -o $@ tools/fvlog_main.cpp -L$(PKG) -lfvlog \
	    -Wl,-rpath,'$$ORIGIN'

tools/fvlog_membench: tools/membench.cu
	$(NVCC) -O3 $(ARCH) -lineinfo -ccbin $(HOSTCXX) -o $@ $<

SORTBENCH_OBJS := $(OBJ)/fv_ctx.o $(OBJ)/radix_sort.o $(OBJ)/prim.o
tools/fvlog_scanbench: tools/scanbench.cu $(OBJ)/fv_ctx.o $(OBJ)/prim.o $(HDRS)
	$(NVCC) $(NVFLAGS) -o $@ $< $(OBJ)/fv_ctx.o $(OBJ)/prim.o -cudart static -lpthread

tools/fvlog_sortbench: tools/sortbench.cu $(SORTBENCH_OBJS) $(HDRS)
	$(NVCC) $(NVFLAGS) -o $@ $< $(SORTBENCH_OBJS) -cudart static -lpthread

clean:
	rm -rf build $(PKG)/libfvlog.so $(PKG)/fvlog tools/fvlog_membench tools/fvlog_sortbench tools/fvlog_scanbench

.PHONY: all clean
