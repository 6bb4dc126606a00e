# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with
# the gpurun snapshot; *.so is git-ignored).
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
CFLAGS  := -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 $(ARCH) -Iinclude
PKG     := paper_2509_24957_b200
SRC_DIR := $(PKG)/csrc
OBJ_DIR := build/obj
LIB     := $(PKG)/libduchess_b200.so
SRCS    := score decide fork kv train mlp mlp_tc tc_linear bw
OBJS    := $(addprefix $(OBJ_DIR)/,$(addsuffix .o,$(SRCS)))
HDRS    := $(SRC_DIR)/common.cuh $(SRC_DIR)/kv_core.cuh $(SRC_DIR)/tc_pair.cuh include/duchess_b200.h

all: $(LIB)

$(OBJ_DIR):
	mkdir -p $@

# decide.cu replays the reference's double arithmetic bit for bit: no FMA contraction.
$(OBJ_DIR)/decide.o: $(SRC_DIR)/decide.cu $(HDRS) | $(OBJ_DIR)
	$(NVCC) $(CFLAGS) --fmad=false -c $< -o $@

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS) | $(OBJ_DIR)
	$(NVCC) $(CFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

ptxas: | $(OBJ_DIR)
	for s in $(SRCS); do $(NVCC) $(CFLAGS) -Xptxas -v -c $(SRC_DIR)/$$s.cu -o /dev/null 2>&1 | grep -E "Function properties|registers|spill" ; done

clean:
	rm -rf build $(LIB)

.PHONY: all clean ptxas
